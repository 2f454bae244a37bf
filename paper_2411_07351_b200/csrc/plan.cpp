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

SubPlan SubPlan::build(int W, int H, int strategy, int block_width) {
    if (W < 1 || H < 1) throw std::invalid_argument("fht2d: image is empty");
    if (strategy != kSimple && strategy != kTweaked) throw std::invalid_argument("unknown split strategy");
    if (block_width < 1 || block_width > 64) throw std::invalid_argument("block width must lie in [1, 64]");
    SubPlan p;
    p.W = W;
    p.H = H;
    p.strategy = strategy;
    p.block_width = block_width;
    p.additions = count_additions_tree(W, H, strategy);

    std::vector<Node> nodes;
    build_tree(nodes, 0, W, 0, strategy, block_width);
    std::map<int, int> shape_of_width;
    int max_upper_depth = -1;
    for (const Node& n : nodes) {
        if (n.w <= block_width) {
            auto it = shape_of_width.find(n.w);
            if (it == shape_of_width.end()) {
                it = shape_of_width.emplace(n.w, static_cast<int>(p.shapes.size())).first;
                p.shapes.push_back(build_shape(n.w, strategy));
            }
            p.blocks.push_back({n.x0, it->second, n.depth});
        } else {
            max_upper_depth = std::max(max_upper_depth, n.depth);
        }
    }
    p.root_is_block = (W <= block_width);
    for (int d = max_upper_depth; d >= 0; --d) {
        UpperLevel lvl;
        lvl.depth = d;
        for (const Node& n : nodes) {
            if (n.depth != d || n.w <= block_width) continue;
            node_ops(n, nodes[static_cast<size_t>(n.child[0])], lvl.ops);
        }
        for (Op& op : lvl.ops) op.r %= H;  // transform.cpp:49
        std::sort(lvl.ops.begin(), lvl.ops.end(), [](const Op& a, const Op& b) { return a.dst < b.dst; });
        p.levels.push_back(std::move(lvl));
    }
    for (const BlockShape& s : p.shapes) {
        p.max_block_width = std::max(p.max_block_width, s.width);
        p.max_halo = std::max(p.max_halo, s.halo);
    }
    return p;
}

std::string SubPlan::describe() const {
    std::ostringstream o;
    o << "{\"W\":" << W << ",\"H\":" << H << ",\"strategy\":" << strategy << ",\"block_width\":" << block_width
      << ",\"root_is_block\":" << (root_is_block ? "true" : "false") << ",\"additions\":" << additions
      << ",\"max_halo\":" << max_halo << ",\"shapes\":[";
    for (size_t i = 0; i < shapes.size(); ++i) {
        const BlockShape& s = shapes[i];
        o << (i ? "," : "") << "{\"width\":" << s.width << ",\"steps\":" << s.depth << ",\"halo\":" << s.halo
          << ",\"ops\":" << s.ops.size() << "}";
    }
    o << "],\"blocks\":" << blocks.size() << ",\"levels\":[";
    for (size_t i = 0; i < levels.size(); ++i)
        o << (i ? "," : "") << "{\"depth\":" << levels[i].depth << ",\"ops\":" << levels[i].ops.size() << "}";
    o << "]}";
    return o.str();
}

}  // namespace fhtb
