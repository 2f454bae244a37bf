// plan.hpp -- integer-exact schedule tables for the FHT2D merge DP.
//
// The reference evaluates the transform by recursion (transform.cpp:35-58):
// split the width (split.hpp:33-48), transform both halves into the other
// ping-pong buffer, then merge every slope t of the node as
//     OUT[t][s] = IN[t0][s] + IN[w0 + t1][(s + r) mod h]
//     t0 = rhu(t (w0-1), w-1), t1 = rhu(t (w1-1), w-1), r = (t - t1) mod h
// with rhu = round_half_up_ratio (split.hpp:53-57).  The SPEC allows any
// evaluation order that is bit-identical.  We evaluate it in a
// few HBM passes, each of which runs several tree levels in shared memory:
//
//  * pass 0, "blocks" (kernel K1): every maximal subtree of width <=
//    block_width.  One CTA computes a whole block for a tile of S rows,
//    reading the input image directly in the quadrant's orientation.  A
//    block's merge schedule depends only on its width: a per-width "shape"
//    table of (dst, a, b, shift) ops in block-local columns (b = -1 carries
//    a leaf one level up).  The rows a tile must load beyond S (the halo)
//    are derived exactly from the tables by propagating the shifts
//    backwards -- never assumed.
//  * passes 1.. "fused upper passes" (kernel K2): the tree above the blocks,
//    cut into bands of at most `pass_levels` levels (by height above the
//    previous pass's output frontier).  Each band node's slopes are cut into
//    tiles of G consecutive slopes; a tile is a small program: load the
//    windows of the frontier columns it depends on (row window offsets and
//    extents derived from the shifts, as for blocks), run its merge ops level
//    by level in shared memory, store its G columns.  The last pass stores
//    the root directly in the reference layout hough[s*W + t].
//
// Pass p writes workspace buffer p % 2 and reads (p-1) % 2: every pass
// consumes exactly the previous pass's frontier (a frontier node with no
// work in a band is carried by a copy tile), so no value is overwritten
// before it is read.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace fhtb {

enum Strategy : int { kSimple = 0, kTweaked = 1 };

// split.hpp:33-48
std::pair<int, int> split_width(int w, int strategy);
// split.hpp:53-57
int64_t round_half_up_ratio(int64_t num, int64_t den);
// oracle.cpp:27-33
uint64_t count_additions_tree(int w, int h, int strategy);

// One gather-add: dst = buf[a] + buf[b] shifted by r (b < 0: copy of a).
struct Op {
    int dst, a, b, r;
};

// K1 shape: the merge schedule of one block width, in block-local columns.
struct BlockShape {
    int width = 0;
    int depth = 0;                 // local depth of the deepest leaf (number of steps)
    int halo = 0;                  // extra input rows a tile of S rows must load
    std::vector<int> step_offset;  // ops of step k (k = 0 is the deepest) at [step_offset[k], step_offset[k+1])
    std::vector<Op> ops;           // r is the UNREDUCED shift t - t1 (< block width)
    std::vector<int> extra;        // per op: rows beyond S the op must produce
};

struct BlockInst {
    int x0, shape, depth;
};

// ---- fused upper passes (K2).  Windows: a value of column c is held for
// rows (s0 + off + i) mod H, i in [0, S + ext).
struct PassLoad {
    int gcol, slot, off, ext;
};
struct PassOp {
    int dst, a, b, ad, bd, ext, pad0, pad1;  // dst[i] = a[i + ad] + b[i + bd], i < S + ext (b < 0: copy)
};
struct PassStore {
    int slot, gcol;
    int slot_hi = -1;  // u16 pair mode: the slot of the root column's upper-half rows
};
struct PassTile {
    int load_beg, load_cnt, step_beg, nsteps, store_beg, store_cnt, nslots, max_ext;
};
// An op of a level-pair program: dst[i] = sum_k slot_k[i + off_k], i < S + ext
// (nterms = 2: one level; 3 or 4: two levels, the intermediate column summed
// in registers instead of stored).
struct PassTerm {
    int slot, off;
};
struct PassOpN {
    int dst, ext, nterms;
    PassTerm term[4];
    int split;  // terms [0, split) form the first child: sum = (first) + (rest), the tree's add order
    int dst_hi = -1;  // u16 pair mode, root ops: the widened upper-half rows go to this slot
};
struct FusedPass {
    int levels = 0;  // tree levels this pass advances (max over its tiles)
    std::vector<PassTile> tiles;
    std::vector<PassLoad> loads;
    std::vector<int> step_offs;  // tile steps: ops [step_offs[step_beg+k], step_offs[step_beg+k+1])
    std::vector<PassOp> ops;
    std::vector<PassStore> stores;
    int max_slots = 0, max_ext = 0, tile_width = 0;
    int64_t loaded_cells = 0;  // sum over tiles of loaded window cells at S = 0 (per-row-tile overhead)
    // The same tiles as a level-pair program (same loads and slots 0..load_cnt):
    // each step advances two levels; an intermediate column read only by the
    // next level is never materialised.  Slots are freed at step boundaries.
    std::vector<PassTile> ptiles;
    std::vector<int> pstep_offs;
    std::vector<PassOpN> pops;
    std::vector<PassStore> pstores;
    int pmax_slots = 0;
    bool root_hi = false;  // the root ops carry dst_hi (u16 pair mode)
};

// The schedule for one working orientation (width W = number of slopes,
// height H = number of shifts).
struct SubPlan {
    int W = 0, H = 0, strategy = kTweaked, block_width = 32;
    std::vector<BlockShape> shapes;
    std::vector<BlockInst> blocks;
    std::vector<FusedPass> passes;  // after K1; passes.back() writes the root
    bool root_is_block = false;
    int max_block_width = 0;
    int max_halo = 0;
    int tree_depth = 0;      // levels of the whole tree (= ceil(log2 W) for Tweaked)
    uint64_t additions = 0;  // count_additions_tree(W, H)

    // root_hi: the root band's level-pair ops get a second output slot (the
    // widening root step of the u16 pair mode)
    static SubPlan build(int W, int H, int strategy, int block_width, int pass_levels, int tile_width,
                         bool root_hi = false);
    std::string describe() const;
};

}  // namespace fhtb

namespace fhtb {
// pattern.cpp:10-30 (Algorithm 2): the slope-t generating pattern of width n.
void build_pattern(int n, int t, int strategy, int* values);
}  // namespace fhtb
