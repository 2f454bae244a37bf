// plan.cpp -- see plan.hpp.  Host-side, integer-exact, built once per
// (size, strategy) and uploaded to the device by the plan object.
#include "plan.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <sstream>
#include <stdexcept>

namespace fhtb {

std::pair<int, int> split_width(int w, int strategy) {
    if (w < 2) throw std::invalid_argument("split: width must be >= 2");
    if (strategy == kSimple) return {w / 2, w - w / 2};  // split.hpp:33-36
    // split.hpp:40-44: first part is the largest power of two strictly below w
    unsigned v = static_cast<unsigned>(w - 1);
    int bw = 0;
    while (v) {
        ++bw;
        v >>= 1;
    }
    const int p = 1 << (bw - 1);
    return {p, w - p};
}

int64_t round_half_up_ratio(int64_t num, int64_t den) {
    if (den < 1) throw std::invalid_argument("round_half_up_ratio: denominator must be positive");
    if (num < 0) throw std::invalid_argument("round_half_up_ratio: numerator must be non-negative");
    return (2 * num + den) / (2 * den);
}

uint64_t count_additions_tree(int w, int h, int strategy) {
    if (w < 1 || h < 1) throw std::invalid_argument("count_additions_tree: sizes must be positive");
    if (w == 1) return 0;
    const auto [w0, w1] = split_width(w, strategy);
    return static_cast<uint64_t>(w) * static_cast<uint64_t>(h) + count_additions_tree(w0, h, strategy) +
           count_additions_tree(w1, h, strategy);
}

namespace {

// pattern.cpp:10-20: split, rescale the slope to both parts (round half up),
// recurse, lift the right part by t - t1.
void pattern_values(int* out, int n, int t, int lift, int strategy) {
    if (n == 1) {
        out[0] = lift;
        return;
    }
    const auto [n0, n1] = split_width(n, strategy);
    const int t0 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (n0 - 1), n - 1));
    const int t1 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (n1 - 1), n - 1));
    pattern_values(out, n0, t0, lift, strategy);
    pattern_values(out + n0, n1, t1, lift + (t - t1), strategy);
}

}  // namespace

void build_pattern(int n, int t, int strategy, int* values) {
    if (n < 1) throw std::invalid_argument("fht2d_pattern: width must be positive");
    if (t < 0 || t >= n) throw std::invalid_argument("fht2d_pattern: slope must lie in [0, n)");
    if (strategy != kSimple && strategy != kTweaked) throw std::invalid_argument("unknown split strategy");
    pattern_values(values, n, t, 0, strategy);
}

namespace {

struct Node {
    int x0, w, depth;
    int child[2];
};

// Recursive split tree of [x0, x0+w) (transform.cpp:41-44), stopping below
// `stop_width` (those nodes are kept as leaves of this tree).
void build_tree(std::vector<Node>& nodes, int x0, int w, int depth, int strategy, int stop_width) {
    const int idx = static_cast<int>(nodes.size());
    nodes.push_back({x0, w, depth, {-1, -1}});
    if (w <= stop_width || w == 1) return;
    const auto [w0, w1] = split_width(w, strategy);
    const int c0 = static_cast<int>(nodes.size());
    build_tree(nodes, x0, w0, depth + 1, strategy, stop_width);
    const int c1 = static_cast<int>(nodes.size());
    build_tree(nodes, x0 + w0, w1, depth + 1, strategy, stop_width);
    nodes[idx].child[0] = c0;
    nodes[idx].child[1] = c1;
}

// The merge ops of one internal node (transform.cpp:46-57), r unreduced.
void node_ops(const Node& n, const Node& left, std::vector<Op>& out) {
    const int w = n.w, w0 = left.w, w1 = n.w - left.w;
    for (int t = 0; t < w; ++t) {
        const int t0 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w0 - 1), w - 1));
        const int t1 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w1 - 1), w - 1));
        out.push_back({n.x0 + t, n.x0 + t0, n.x0 + w0 + t1, t - t1});
    }
}

BlockShape build_shape(int wb, int strategy) {
    BlockShape sh;
    sh.width = wb;
    std::vector<Node> nodes;
    build_tree(nodes, 0, wb, 0, strategy, 0);
    int dmax = 0;
    for (const Node& n : nodes) dmax = std::max(dmax, n.depth);
    sh.depth = dmax;
    // Top-down step lists: step ld (0 = block root) writes the depth-ld values.
    std::vector<std::vector<Op>> by_depth(static_cast<size_t>(dmax));
    for (int ld = 0; ld < dmax; ++ld) {
        for (const Node& n : nodes) {
            if (n.child[0] >= 0 && n.depth == ld) node_ops(n, nodes[static_cast<size_t>(n.child[0])], by_depth[ld]);
            if (n.child[0] < 0 && n.depth <= ld) by_depth[ld].push_back({n.x0, n.x0, -1, 0});  // carry a leaf
        }
        std::sort(by_depth[ld].begin(), by_depth[ld].end(), [](const Op& a, const Op& b) { return a.dst < b.dst; });
        if (static_cast<int>(by_depth[ld].size()) != wb) throw std::logic_error("block step does not cover every column");
    }
    // Backward need propagation: rows beyond S each value must cover so that
    // the block root's rows [0, S) are exact.  need_out = 0 at the root.
    std::vector<std::vector<int>> extra(static_cast<size_t>(dmax));
    std::vector<int> need_out(static_cast<size_t>(wb), 0);
    for (int ld = 0; ld < dmax; ++ld) {
        std::vector<int> need_in(static_cast<size_t>(wb), 0);
        for (const Op& op : by_depth[ld]) {
            const int e = need_out[static_cast<size_t>(op.dst)];
            extra[ld].push_back(e);
            need_in[static_cast<size_t>(op.a)] = std::max(need_in[static_cast<size_t>(op.a)], e);
            if (op.b >= 0) need_in[static_cast<size_t>(op.b)] = std::max(need_in[static_cast<size_t>(op.b)], e + op.r);
        }
        need_out = need_in;
    }
    sh.halo = 0;
    for (int v : need_out) sh.halo = std::max(sh.halo, v);
    // Emit deepest step first (execution order).
    sh.step_offset.push_back(0);
    for (int ld = dmax - 1; ld >= 0; --ld) {
        for (size_t k = 0; k < by_depth[ld].size(); ++k) {
            sh.ops.push_back(by_depth[ld][k]);
            sh.extra.push_back(extra[ld][k]);
        }
        sh.step_offset.push_back(static_cast<int>(sh.ops.size()));
    }
    return sh;
}

}  // namespace

namespace {

// One fused tile: the slopes [ta, tb) of band node X, whose inputs are the
// frontier nodes below it.  Appends the program to `ps`.
void build_tile(const std::vector<Node>& nodes, const std::vector<char>& front, const std::vector<int>& height,
                int X, int ta, int tb, int H, FusedPass& ps) {
    struct Entry {
        int lo = 0, hi = 0;  // window rows [s0+lo, s0+hi+S): ext = hi - lo
        int slot = -1;
        int last_use = -1;   // last step reading it
        bool seen = false;
    };
    // Entries per node: local column -> Entry (only needed columns).
    std::vector<std::vector<Entry>> ent(nodes.size());
    std::vector<int> order;  // nodes of the tile program, parents before children
    auto touch = [&](int n) {
        if (ent[static_cast<size_t>(n)].empty()) {
            ent[static_cast<size_t>(n)].resize(static_cast<size_t>(nodes[static_cast<size_t>(n)].w));
            order.push_back(n);
        }
    };
    touch(X);
    for (int t = ta; t < tb; ++t) {
        Entry& e = ent[static_cast<size_t>(X)][static_cast<size_t>(t)];
        e.seen = true;
        e.lo = 0;
        e.hi = 0;
    }
    for (size_t qi = 0; qi < order.size(); ++qi) {
        const int n = order[qi];
        // All consumers of n are known now: align its window starts down to a
        // multiple of 4 rows, so every a-operand and destination of the
        // kernel's 16-byte vector merges is aligned (only b is shifted).
        for (Entry& e : ent[static_cast<size_t>(n)])
            if (e.seen) e.lo &= ~3;
        if (front[static_cast<size_t>(n)]) continue;  // input node
        const Node& nd = nodes[static_cast<size_t>(n)];
        const int c0 = nd.child[0], c1 = nd.child[1];
        const int w = nd.w, w0 = nodes[static_cast<size_t>(c0)].w, w1 = w - w0;
        touch(c0);
        touch(c1);
        for (int t = 0; t < w; ++t) {
            const Entry& e = ent[static_cast<size_t>(n)][static_cast<size_t>(t)];
            if (!e.seen) continue;
            const int t0 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w0 - 1), w - 1));
            const int t1 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w1 - 1), w - 1));
            const int r = (t - t1) % H;
            Entry& a = ent[static_cast<size_t>(c0)][static_cast<size_t>(t0)];
            Entry& b = ent[static_cast<size_t>(c1)][static_cast<size_t>(t1)];
            if (!a.seen) a.lo = e.lo, a.hi = e.hi, a.seen = true;
            a.lo = std::min(a.lo, e.lo);
            a.hi = std::max(a.hi, e.hi);
            if (!b.seen) b.lo = e.lo + r, b.hi = e.hi + r, b.seen = true;
            b.lo = std::min(b.lo, e.lo + r);
            b.hi = std::max(b.hi, e.hi + r);
        }
    }
    // Steps by height above the frontier; last use of every entry.
    const int hx = height[static_cast<size_t>(X)];
    std::vector<std::vector<int>> step_nodes(static_cast<size_t>(std::max(hx, 0)));
    for (int n : order)
        if (!front[static_cast<size_t>(n)]) step_nodes[static_cast<size_t>(height[static_cast<size_t>(n)] - 1)].push_back(n);
    for (int j = 0; j < hx; ++j)
        for (int n : step_nodes[static_cast<size_t>(j)]) {
            const Node& nd = nodes[static_cast<size_t>(n)];
            const int c0 = nd.child[0], c1 = nd.child[1];
            const int w = nd.w, w0 = nodes[static_cast<size_t>(c0)].w, w1 = w - w0;
            for (int t = 0; t < w; ++t) {
                if (!ent[static_cast<size_t>(n)][static_cast<size_t>(t)].seen) continue;
                const int t0 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w0 - 1), w - 1));
                const int t1 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w1 - 1), w - 1));
                ent[static_cast<size_t>(c0)][static_cast<size_t>(t0)].last_use = j;
                ent[static_cast<size_t>(c1)][static_cast<size_t>(t1)].last_use = j;
            }
        }
    // Slot allocation: loads first, then each step's outputs from slots freed
    // by earlier steps (a slot is never reused within the step that frees it).
    PassTile tile{};
    tile.load_beg = static_cast<int>(ps.loads.size());
    tile.step_beg = static_cast<int>(ps.step_offs.size());
    tile.nsteps = hx;
    tile.store_beg = static_cast<int>(ps.stores.size());
    int next_slot = 0, max_ext = 0;
    std::vector<int> free_slots;
    for (int n : order) {
        if (!front[static_cast<size_t>(n)]) continue;
        const Node& nd = nodes[static_cast<size_t>(n)];
        for (int t = 0; t < nd.w; ++t) {
            Entry& e = ent[static_cast<size_t>(n)][static_cast<size_t>(t)];
            if (!e.seen) continue;
            e.slot = next_slot++;
            ps.loads.push_back({nd.x0 + t, e.slot, e.lo, e.hi - e.lo});
            ps.loaded_cells += e.hi - e.lo;
            max_ext = std::max(max_ext, e.hi - e.lo);
        }
    }
    tile.load_cnt = static_cast<int>(ps.loads.size()) - tile.load_beg;
    std::vector<std::pair<int, int>> live;  // (node, col) computed so far, for freeing
    for (int n : order)
        if (front[static_cast<size_t>(n)])
            for (int t = 0; t < nodes[static_cast<size_t>(n)].w; ++t)
                if (ent[static_cast<size_t>(n)][static_cast<size_t>(t)].seen) live.push_back({n, t});
    for (int j = 0; j < hx; ++j) {
        ps.step_offs.push_back(static_cast<int>(ps.ops.size()));
        for (int n : step_nodes[static_cast<size_t>(j)]) {
            const Node& nd = nodes[static_cast<size_t>(n)];
            const int c0 = nd.child[0], c1 = nd.child[1];
            const int w = nd.w, w0 = nodes[static_cast<size_t>(c0)].w, w1 = w - w0;
            for (int t = 0; t < w; ++t) {
                Entry& e = ent[static_cast<size_t>(n)][static_cast<size_t>(t)];
                if (!e.seen) continue;
                const int t0 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w0 - 1), w - 1));
                const int t1 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(t) * (w1 - 1), w - 1));
                const int r = (t - t1) % H;
                const Entry& a = ent[static_cast<size_t>(c0)][static_cast<size_t>(t0)];
                const Entry& b = ent[static_cast<size_t>(c1)][static_cast<size_t>(t1)];
                if (free_slots.empty()) {
                    e.slot = next_slot++;
                } else {
                    e.slot = free_slots.back();
                    free_slots.pop_back();
                }
                PassOp op{};
                op.dst = e.slot;
                op.a = a.slot;
                op.b = b.slot;
                op.ad = e.lo - a.lo;
                op.bd = e.lo + r - b.lo;
                op.ext = e.hi - e.lo;
                if (op.ad < 0 || op.bd < 0 || op.ad + op.ext > a.hi - a.lo || op.bd + op.ext > b.hi - b.lo)
                    throw std::logic_error("fused tile window derivation failed");
                ps.ops.push_back(op);
                max_ext = std::max(max_ext, op.ext);
                live.push_back({n, t});
            }
        }
        // free the slots whose last consumer was this step (usable from step j+1)
        std::vector<std::pair<int, int>> keep;
        for (auto [n, t] : live) {
            const Entry& e = ent[static_cast<size_t>(n)][static_cast<size_t>(t)];
            if (n != X && e.last_use == j)
                free_slots.push_back(e.slot);
            else
                keep.push_back({n, t});
        }
        live.swap(keep);
    }
    ps.step_offs.push_back(static_cast<int>(ps.ops.size()));
    const Node& xn = nodes[static_cast<size_t>(X)];
    for (int t = ta; t < tb; ++t) ps.stores.push_back({ent[static_cast<size_t>(X)][static_cast<size_t>(t)].slot, xn.x0 + t});
    tile.store_cnt = tb - ta;
    tile.nslots = next_slot;
    tile.max_ext = max_ext;
    ps.max_slots = std::max(ps.max_slots, next_slot);
    ps.max_ext = std::max(ps.max_ext, max_ext);
    ps.tiles.push_back(tile);

    // ---- the level-pair program of the same tile (steps 2g, 2g+1 fused)
    PassTile pt = tile;
    pt.step_beg = static_cast<int>(ps.pstep_offs.size());
    pt.nsteps = (hx + 1) / 2;
    pt.store_beg = static_cast<int>(ps.pstores.size());
    std::vector<std::vector<int>> pslot(nodes.size());
    for (int n : order) pslot[static_cast<size_t>(n)].assign(static_cast<size_t>(nodes[static_cast<size_t>(n)].w), -1);
    for (int n : order)
        if (front[static_cast<size_t>(n)])
            for (int t = 0; t < nodes[static_cast<size_t>(n)].w; ++t)
                pslot[static_cast<size_t>(n)][static_cast<size_t>(t)] = ent[static_cast<size_t>(n)][static_cast<size_t>(t)].slot;
    int pnext = tile.load_cnt;
    std::vector<int> pfree;
    std::vector<int> phi(static_cast<size_t>(nodes[static_cast<size_t>(X)].w), -1);  // root upper-row slots
    std::vector<std::pair<int, int>> plive;
    for (int n : order)
        if (front[static_cast<size_t>(n)])
            for (int t = 0; t < nodes[static_cast<size_t>(n)].w; ++t)
                if (ent[static_cast<size_t>(n)][static_cast<size_t>(t)].seen) plive.push_back({n, t});
    auto step_of = [&](int n) { return front[static_cast<size_t>(n)] ? -1 : height[static_cast<size_t>(n)] - 1; };
    for (int gs = 0; gs < hx; gs += 2) {
        const int ge = std::min(hx, gs + 2) - 1;
        ps.pstep_offs.push_back(static_cast<int>(ps.pops.size()));
        for (int j = gs; j <= ge; ++j)
            for (int n : step_nodes[static_cast<size_t>(j)]) {
                const Node& nd = nodes[static_cast<size_t>(n)];
                for (int t = 0; t < nd.w; ++t) {
                    const Entry& e = ent[static_cast<size_t>(n)][static_cast<size_t>(t)];
                    if (!e.seen) continue;
                    // stored, or read after this step: materialise; else the
                    // next level of the pair sums its terms itself
                    if (n != X && e.last_use <= ge) continue;
                    PassOpN op{};
                    op.ext = e.hi - e.lo;
                    // terms of (node, col) at a row shift: a child made earlier in
                    // this step is expanded into its own two terms
                    auto add_terms = [&](auto&& self, int m, int c, int shift, bool expand) -> void {
                        if (!expand) {
                            const Entry& ce = ent[static_cast<size_t>(m)][static_cast<size_t>(c)];
                            const int slot = pslot[static_cast<size_t>(m)][static_cast<size_t>(c)];
                            const int off = e.lo + shift - ce.lo;
                            if (op.nterms >= 4 || slot < 0 || off < 0 || off + op.ext > ce.hi - ce.lo)
                                throw std::logic_error("level-pair program derivation failed");
                            op.term[op.nterms++] = {slot, off};
                            return;
                        }
                        const Node& md = nodes[static_cast<size_t>(m)];
                        const int w = md.w, w0 = nodes[static_cast<size_t>(md.child[0])].w, w1 = w - w0;
                        const int t0 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(c) * (w0 - 1), w - 1));
                        const int t1 = static_cast<int>(round_half_up_ratio(static_cast<int64_t>(c) * (w1 - 1), w - 1));
                        const int r = (c - t1) % H;
                        self(self, md.child[0], t0, shift, step_of(md.child[0]) >= gs && m == n);
                        if (m == n) op.split = op.nterms;  // terms of the first child: the add order
                        self(self, md.child[1], t1, shift + r, step_of(md.child[1]) >= gs && m == n);
                    };
                    add_terms(add_terms, n, t, 0, true);
                    // A stored column prefers a freed slot of index == its slope mod 8:
                    // the root store reads 16-32 of them at one row offset, and with
                    // every residue equally often (slot stride L, L/4 odd) the reads
                    // spread evenly over the shared-memory banks.
                    auto take = [&](int want) {
                        if (pfree.empty()) return pnext++;
                        size_t pick = pfree.size() - 1;
                        if (want >= 0)
                            for (size_t k = pfree.size(); k-- > 0;)
                                if ((pfree[k] & 7) == want) {
                                    pick = k;
                                    break;
                                }
                        const int sl = pfree[pick];
                        pfree.erase(pfree.begin() + static_cast<std::ptrdiff_t>(pick));
                        return sl;
                    };
                    const int want = n == X ? (t - ta) & 7 : -1;
                    op.dst = take(want);
                    pslot[static_cast<size_t>(n)][static_cast<size_t>(t)] = op.dst;
                    if (ps.root_hi && X == 0 && n == X) {  // the widened root's upper rows
                        op.dst_hi = take(want);
                        phi[static_cast<size_t>(t)] = op.dst_hi;
                    }
                    ps.pops.push_back(op);
                    plive.push_back({n, t});
                }
            }
        // free what was last read in this step (reusable from the next step)
        std::vector<std::pair<int, int>> keep;
        for (auto [n, t] : plive) {
            const Entry& e = ent[static_cast<size_t>(n)][static_cast<size_t>(t)];
            if (n != X && e.last_use <= ge)
                pfree.push_back(pslot[static_cast<size_t>(n)][static_cast<size_t>(t)]);
            else
                keep.push_back({n, t});
        }
        plive.swap(keep);
    }
    ps.pstep_offs.push_back(static_cast<int>(ps.pops.size()));
    for (int t = ta; t < tb; ++t)
        ps.pstores.push_back({pslot[static_cast<size_t>(X)][static_cast<size_t>(t)], xn.x0 + t, phi[static_cast<size_t>(t)]});
    pt.nslots = pnext;
    ps.pmax_slots = std::max(ps.pmax_slots, pnext);
    ps.ptiles.push_back(pt);
}

}  // namespace

SubPlan SubPlan::build(int W, int H, int strategy, int block_width, int pass_levels, int tile_width, bool root_hi) {
    if (W < 1 || H < 1) throw std::invalid_argument("fht2d: image is empty");
    if (strategy != kSimple && strategy != kTweaked) throw std::invalid_argument("unknown split strategy");
    if (block_width < 1 || block_width > 64) throw std::invalid_argument("block width must lie in [1, 64]");
    if (pass_levels < 1 || pass_levels > 8) throw std::invalid_argument("pass levels must lie in [1, 8]");
    if (tile_width < 1) throw std::invalid_argument("tile width must be positive");
    SubPlan p;
    p.W = W;
    p.H = H;
    p.strategy = strategy;
    p.block_width = block_width;
    p.additions = count_additions_tree(W, H, strategy);

    std::vector<Node> nodes;
    build_tree(nodes, 0, W, 0, strategy, block_width);
    std::map<int, int> shape_of_width;
    std::vector<char> front(nodes.size(), 0);
    for (size_t i = 0; i < nodes.size(); ++i) {
        const Node& n = nodes[i];
        if (n.w <= block_width) {
            auto it = shape_of_width.find(n.w);
            if (it == shape_of_width.end()) {
                it = shape_of_width.emplace(n.w, static_cast<int>(p.shapes.size())).first;
                p.shapes.push_back(build_shape(n.w, strategy));
            }
            p.blocks.push_back({n.x0, it->second, n.depth});
            front[i] = 1;
            p.tree_depth = std::max(p.tree_depth, n.depth + p.shapes[static_cast<size_t>(it->second)].depth);
        }
    }
    p.root_is_block = (W <= block_width);
    for (const BlockShape& s : p.shapes) {
        p.max_block_width = std::max(p.max_block_width, s.width);
        p.max_halo = std::max(p.max_halo, s.halo);
    }
    // Parent pointers (nodes are in preorder: children follow their parent).
    std::vector<int> parent(nodes.size(), -1);
    for (size_t i = 0; i < nodes.size(); ++i)
        for (int c : nodes[i].child)
            if (c >= 0) parent[static_cast<size_t>(c)] = static_cast<int>(i);
    // Bands of <= pass_levels levels above the current frontier.
    while (!front[0]) {
        std::vector<char> below(nodes.size(), 0);
        for (size_t i = 1; i < nodes.size(); ++i) {
            const size_t pa = static_cast<size_t>(parent[i]);
            below[i] = below[pa] || front[pa];
        }
        std::vector<int> height(nodes.size(), 0);
        for (size_t ii = nodes.size(); ii-- > 0;) {
            if (below[ii] || front[ii]) continue;
            const Node& n = nodes[ii];
            height[ii] = 1 + std::max(height[static_cast<size_t>(n.child[0])], height[static_cast<size_t>(n.child[1])]);
        }
        const int U = height[0];
        const int npass = (U + pass_levels - 1) / pass_levels;
        const int k = (U + npass - 1) / npass;
        std::vector<char> nfront(nodes.size(), 0);
        FusedPass ps;
        ps.tile_width = tile_width;
        ps.root_hi = root_hi;
        for (size_t i = 0; i < nodes.size(); ++i) {
            if (below[i]) continue;
            const bool top = (i == 0) || height[static_cast<size_t>(parent[i])] > k;
            if (height[i] > k || !top) continue;
            nfront[i] = 1;
            ps.levels = std::max(ps.levels, height[i]);
            const int w = nodes[i].w;
            for (int ta = 0; ta < w; ta += tile_width)
                build_tile(nodes, front, height, static_cast<int>(i), ta, std::min(w, ta + tile_width), H, ps);
        }
        p.passes.push_back(std::move(ps));
        front.swap(nfront);
    }
    return p;
}

std::string SubPlan::describe() const {
    std::ostringstream o;
    o << "{\"W\":" << W << ",\"H\":" << H << ",\"strategy\":" << strategy << ",\"block_width\":" << block_width
      << ",\"root_is_block\":" << (root_is_block ? "true" : "false") << ",\"additions\":" << additions
      << ",\"tree_depth\":" << tree_depth << ",\"max_halo\":" << max_halo << ",\"shapes\":[";
    for (size_t i = 0; i < shapes.size(); ++i) {
        const BlockShape& s = shapes[i];
        o << (i ? "," : "") << "{\"width\":" << s.width << ",\"steps\":" << s.depth << ",\"halo\":" << s.halo
          << ",\"ops\":" << s.ops.size() << "}";
    }
    o << "],\"blocks\":" << blocks.size() << ",\"passes\":[";
    for (size_t i = 0; i < passes.size(); ++i) {
        const FusedPass& f = passes[i];
        o << (i ? "," : "") << "{\"levels\":" << f.levels << ",\"tiles\":" << f.tiles.size()
          << ",\"tile_width\":" << f.tile_width << ",\"loads\":" << f.loads.size() << ",\"ops\":" << f.ops.size()
          << ",\"stores\":" << f.stores.size() << ",\"max_slots\":" << f.max_slots << ",\"max_ext\":" << f.max_ext
          << ",\"loaded_ext_cells\":" << f.loaded_cells << "}";
    }
    o << "]}";
    return o.str();
}

}  // namespace fhtb
