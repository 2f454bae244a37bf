// plan.hpp -- integer-exact schedule tables for the FHT2D merge DP.
//
// The reference evaluates the transform by recursion (transform.cpp:35-58):
// split the width (split.hpp:33-48), transform both halves into the other
// ping-pong buffer, then merge every slope t of the node as
//     OUT[t][s] = IN[t0][s] + IN[w0 + t1][(s + r) mod h]
//     t0 = rhu(t (w0-1), w-1), t1 = rhu(t (w1-1), w-1), r = (t - t1) mod h
// with rhu = round_half_up_ratio (split.hpp:53-57).  The SPEC allows any
// evaluation order that is bit-identical; we evaluate it
// level-order on the GPU:
//
//  * "blocks": every maximal subtree of width <= block_width.  One CTA
//    computes a whole block for a tile of S rows in shared memory (kernel
//    K1), reading the input image in the quadrant's orientation.  A block's
//    merge schedule depends only on its width, so it is a per-width "shape"
//    table of (dst, a, b, shift) ops in block-local columns, with b = -1
//    meaning "carry a leaf column one level up".  The rows a tile must load
//    (the halo) are derived exactly from the tables by propagating the
//    shifts backwards -- never assumed.
//  * "upper levels": every node wider than block_width is one gather-add op
//    per slope in an HBM/L2 ping-pong pass (kernel K2) per tree depth.  The
//    root level (depth 0) is fused with the store into the reference output
//    layout (kernel K3).
//
// A node at depth d writes buffer d % 2 (exactly the reference's out/tmp
// alternation, transform.cpp:42-44), so blocks of different depths and
// upper nodes of different depths never overwrite a value before its parent
// reads it.
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
    std::vector<Op> ops;           // r is the UNREDUCED shift t - t1; `extra` rows packed in r's high half
    std::vector<int> extra;        // per op: rows beyond S the op must produce
};

struct BlockInst {
    int x0, shape, depth;
};

struct UpperLevel {
    int depth;
    std::vector<Op> ops;  // global columns, r reduced mod h
};

// The schedule for one working orientation (width W = number of slopes,
// height H = number of shifts).
struct SubPlan {
    int W = 0, H = 0, strategy = kTweaked, block_width = 32;
    std::vector<BlockShape> shapes;
    std::vector<BlockInst> blocks;
    std::vector<UpperLevel> levels;  // ordered deepest first; levels.back() is the root (depth 0) if root is upper
    bool root_is_block = false;
    int max_block_width = 0;
    int max_halo = 0;
    uint64_t additions = 0;  // count_additions_tree(W, H)

    static SubPlan build(int W, int H, int strategy, int block_width);
    std::string describe() const;
};

}  // namespace fhtb
