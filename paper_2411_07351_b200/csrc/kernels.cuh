// kernels.cuh -- launch interface of the sm_100a FHT2D merge kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fhtb {

enum DType : int { kU8 = 0, kI32 = 1, kI64 = 2, kF32 = 3 };

// Quadrant codes (reference QuadrantSet order, quadrants.hpp:23-28):
//   0 horiz_pos = fht2d(I)            COLS[x][y] = I[y][x]
//   1 horiz_neg = fht2d(flipH(I))     COLS[x][y] = I[y][w-1-x]
//   2 vert_pos  = fht2d(I^T)          COLS[x][y] = I[x][y]
//   3 vert_neg  = fht2d(flipH(I^T))   COLS[x][y] = I[h-1-x][y]
struct QuadSet {
    int code[4];
    int n;
};

// Output of the root level.  ptr[q] is the quadrant-q Hough image of image
// 0; image i is at ptr[q] + i * img_stride elements.  layout 0 is the
// reference layout hough[s * W + t] (transform.cpp:80-83); layout 1 is the
// native slope-major layout hough[t * H + s].
struct OutDesc {
    void* ptr[4];
    long long img_stride;
    int layout;
    int dtype;
    // slope-major (native) layout only: slopes [peer_c0, peer_c1) are also
    // stored to peer + (t - peer_c0) * H -- another GPU's buffer mapped over
    // NVLink (the root split's exchange, fused into the child's last pass)
    void* peer;
    int peer_c0, peer_c1;
};

// Per K1 shape header (8 ints): width, nsteps, op_base, step_base, halo.
struct ShapeHdr {
    int width, nsteps, op_base, step_base, halo, pad0, pad1, pad2;
};

// Device tables of one fused upper pass (see plan.hpp FusedPass).
struct PassTileDev {
    int load_beg, load_cnt, step_beg, nsteps, store_beg, store_cnt, nslots, max_ext;
};
struct PassOpDev {
    int dst, a, b, ad, bd, ext, pad0, pad1;
};
struct PassDev {
    const PassTileDev* tiles;
    const int4* loads;  // gcol, slot, off, ext
    const int* step_offs;
    const PassOpDev* ops;
    const int4* bops;    // ops baked for 4-byte accumulators: shared byte offsets {dst, a, b|M, rows}
    const int2* stores;  // slot, gcol
    int ntiles;
    int S;       // rows per row tile
    int L;       // smem row capacity of a slot (>= S + max_ext, odd)
    int max_slots;
    int max_tile_ops;  // most merge ops in one tile (staged in shared memory)
    int bulk;          // window runs by TMA bulk copies (set per launch)
    int pairs;         // the tables are level-pair programs (bops: 2 records per op)
    // u16 pair mode root band, double-buffered windows (k2_pair_pipe): the same
    // ops / stores with every load-space slot s < tile.load_cnt moved to
    // s + pipe_delta (the second window buffer); pipe_delta = 0: no such tables
    const int4* bops1;
    const int2* stores1;
    int pipe_delta, pipe_loads;  // slot offset of the second buffer, its size (max load_cnt)
    int tile_nc_max;             // most stored slopes of one tile
    // TMA windows for k2_pair_pipe (tma = 1; one row tile, s0 = 0): per load,
    // {gcol, bulk dst byte, bulk src word, bulk words}, {small dst byte, small
    // src word (wraps mod H), small count, 0}; dst bytes are relative to the
    // window buffer; tbops / tbops1 = bops / bops1 with every window term
    // moved by its window's alignment residue
    int tma;
    const int4* twin;
    const int4* tbops;
    const int4* tbops1;
    // TMA windows in k2_pass (ktma = 1; level-pair programs, 4-byte
    // accumulators): per op the window index each term reads (4 x u8, 0xff
    // none); the stores with bit 30 of the column set read a window
    int ktma;
    const int* kwslots;
    const int2* kwstores;
    // timing probe (FHT_K2_PROBE, debug only; results are wrong when set):
    // bit 0 skips the merges, bit 1 the root store, bit 2 the window copies
    // after the first slot (k2_pair_pipe)
    int probe;
};

struct GroupLaunch {
    // image
    const void* img;
    int in_dtype;
    int img_w, img_h;
    long long img_pitch;  // elements between image rows (>= img_w)
    long long img_stride;
    int img0;      // first image of this chunk
    int nimg;      // images in this chunk
    QuadSet qs;
    // working orientation
    int W, H, ld;
    int acc_dtype;
    // K1
    int S;
    int nblocks;        // generic (table-driven) blocks
    const int4* blocks;
    int nby;            // width-32 Brady-Yong blocks for the specialised K1P (4-byte accumulators)
    const int* by_x0;
    cudaStream_t aux_stream;  // plan-owned stream for the concurrent generic-block K1 (may be null)
    cudaEvent_t ev_fork, ev_join;
    // held around each event record + stream wait pair: a plan (and so its
    // aux stream and events) may be executed by several host threads at
    // once, and a wait must see the record of its own call (std::mutex*)
    void* fork_mu;
    // int64 plans whose pass-0 sums fit int32 (32 * max|v| < 2^31): K1 and
    // K1P accumulate in int32 and widen as they store the block roots
    int k1_acc32 = 0;
    int k1p_variant;    // 5 (default): 4, with levels 1-2 reading the staged u8 columns directly
                        // (no leaf tile) when the input is staged; 4: levels 1-2 in registers,
                        // 3-5 rows interleaved over lanes, the root stored from registers;
                        // 3: root via shared memory; 2: levels 3-5 with 4 rows per lane;
                        // 0: all levels in shared memory
    int pdl;            // programmatic dependent launch of the stream-ordered kernels
    int k2_bulk;        // K2 aligned window runs by cp.async.bulk (TMA) instead of 16-byte cp.async
    int k2_scalar;      // 1 (default): K2 merge rows interleaved over lanes; 0: 4 rows per lane (int4)
    const ShapeHdr* shapes;
    const int* step_offs;
    const PassOpDev* k1_ops;  // per-shape ops, slots pre-offset by buffer parity
    const int4* k1_bops;      // the same, baked into shared byte offsets (4-byte accumulators)
    int k1_max_ops, k1_max_steps, k1_max_width, k1_sr;
    bool root_is_block;
    // fused upper passes (K2), in execution order; the last writes the root
    int npasses;
    const PassDev* passes;
    // workspace: per slot nbuf (1 or 2) W x ld buffers
    void* ws;
    int nbuf;
    OutDesc out;
    // u8 staging for K1P (null: K1P reads the image itself): per image, the
    // working columns of the horizontal quadrants (image columns, at
    // stage_t) and/or of the vertical ones (image rows, at stage_p), W
    // columns of stage_pitch bytes each, rows past H wrapped
    // u16 pair mode (0: off): workspace words hold rows (j, j + pm_D);
    // K1/K1P/K2 run one row tile of pm_D words, K2's root step widens to 32 bits
    int pm_D;
    int k1p_pair576;  // pair mode: K1P on 576 threads (one round of level-1/2 items)
    int k1p_576;      // K1P variant 5 outside the pair mode on 576 threads (same reason)
    unsigned char* stage;
    long long stage_pitch, stage_img;
    long long stage_t, stage_p;  // byte offsets inside an image's stage (-1: not staged)
};

size_t k1_smem_bytes(int acc_dtype, int max_width, int sr, int max_ops, int max_steps);
size_t k2_smem_bytes(int acc_dtype, int max_slots, int L, int max_tile_ops);
// Launch every kernel of one orientation group / chunk on `stream`.
// Returns the number of kernel launches, or -1 on an unsupported type combination.
// `hook(ctx, kind)` (optional) runs after each launch; kind 1 = K1 (generic
// blocks), 4 = K1P (width-32 Brady-Yong blocks), 2 = K2 (fused upper pass),
// 3 = K2 writing the root.
typedef void (*LaunchHook)(void* ctx, int kind);
int launch_group(const GroupLaunch& g, cudaStream_t stream, LaunchHook hook = nullptr, void* ctx = nullptr);

// Root merge of a width-W node from its children's slope-major column ranges
// (left columns [left_first, ...), right columns [right_first, ...)), output
// slopes [t_beg, t_end); d_ops[t] = (t, t0, t1, r).  Returns -1 on a bad type pair.
int launch_merge_root(const int4* d_ops, const void* left, int left_first, const void* right, int right_first,
                      int W, int H, int t_beg, int t_end, void* out, int acc, int outd, int layout, cudaStream_t st);

// Device max |v| over n int32/int64 values into *d_max (must be zeroed).
void launch_absmax(const void* d_in, int dtype, long long n, unsigned long long* d_max, cudaStream_t stream);

}  // namespace fhtb
