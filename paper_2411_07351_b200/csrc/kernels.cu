// kernels.cu -- sm_100a kernels for the FHT2D merge DP (transform.cpp:35-58).
//
// K1 k1_blocks : load an input tile in the quadrant's orientation straight
//                from the row-major image (no flip / transpose copies,
//                quadrants.cpp:7-21) and run every level of one block
//                (maximal subtree of width <= block_width) in shared memory.
// K2 k2_level  : one upper merge level, OUT[t] = IN[a] + rot(IN[b], r), as a
//                coalesced, vectorised HBM/L2 ping-pong pass.
// K3 k3_root   : the root level fused with the store into the reference
//                layout hough[s*W + t] (transform.cpp:80-83) through an smem
//                transpose, optionally widening to int64.
// The path is a gather-add: no contraction, so no tensor cores; every kernel
// is bound by HBM (or L2) bandwidth.  See DESIGN.md for the roofline model.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels.cuh"

namespace fhtb {

namespace {

constexpr int kThreads = 256;

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ int wrap_once(int j, int H) { return j >= H ? j - H : j; }

__device__ __forceinline__ int wrap_any(int j, int H) {
    if (j >= H) j -= H;
    if (j >= H) j %= H;
    return j;
}

// Element (working column x, working row y) of quadrant q of a row-major image.
template <class In>
__device__ __forceinline__ In load_quadrant(const In* __restrict__ im, int q, int x, int y, int img_w,
                                            int img_h) {
    switch (q) {
        case 0: return im[(size_t)y * img_w + x];
        case 1: return im[(size_t)y * img_w + (img_w - 1 - x)];
        case 2: return im[(size_t)x * img_w + y];
        default: return im[(size_t)(img_h - 1 - x) * img_w + y];
    }
}

template <class T>
__device__ __forceinline__ T from_bits(int v) {
    if constexpr (std::is_same<T, float>::value) return __int_as_float(v);
    else return static_cast<T>(v);
}
template <class T>
__device__ __forceinline__ int to_bits(T v) {
    if constexpr (std::is_same<T, float>::value) return __float_as_int(v);
    else return static_cast<int>(v);
}

__device__ __forceinline__ size_t k1_ops_offset_dev(size_t esz, int max_width, int sr) {
    return (2 * static_cast<size_t>(max_width) * sr * esz + 15) / 16 * 16;
}

// ------------------------------------------------------------------- K1
// grid: x = row tile (S rows), y = block, z = slot (image * nq + quadrant idx)
template <class In, class Acc, class Out>
__global__ void __launch_bounds__(kThreads) k1_blocks(
    const In* __restrict__ img, int img_w, int img_h, long long img_stride, int img0, QuadSet qs, int W, int H,
    int ld, int S, const int4* __restrict__ blocks, const ShapeHdr* __restrict__ shapes,
    const int* __restrict__ step_offs, const int4* __restrict__ ops, int max_width, int sr, int max_ops,
    Acc* __restrict__ ws, int nbuf, bool root_is_block, OutDesc out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* buf0 = reinterpret_cast<Acc*>(smem_raw);
    Acc* buf1 = buf0 + (size_t)max_width * sr;
    int4* sops = reinterpret_cast<int4*>(smem_raw + k1_ops_offset_dev(sizeof(Acc), max_width, sr));
    int* soffs = reinterpret_cast<int*>(sops + max_ops);

    const int tid = threadIdx.x;
    const int4 blk = blocks[blockIdx.y];
    const int x0 = blk.x;
    const ShapeHdr hdr = shapes[blk.y];
    const int wb = hdr.width, nsteps = hdr.nsteps;
    const int R = S + hdr.halo;
    const int nops_total = wb * nsteps;
    for (int k = tid; k < nops_total; k += kThreads) sops[k] = ops[hdr.op_base + k];
    for (int k = tid; k <= nsteps; k += kThreads) soffs[k] = step_offs[hdr.step_base + k];

    const int slot = blockIdx.z;
    const int nq = qs.n;
    const int img_i = img0 + slot / nq;
    const int q = qs.code[slot % nq];
    const In* __restrict__ im = img + (size_t)img_i * img_stride;
    const int s0 = blockIdx.x * S;

    // Load the tile: values of depth `nsteps` (the leaves) into buf[nsteps & 1].
    Acc* lbuf = (nsteps & 1) ? buf1 : buf0;
    const int cells = wb * R;
    if (q < 2) {  // working column = image column: contiguous along c
        for (int k = tid; k < cells; k += kThreads) {
            const int c = k % wb, i = k / wb;
            const int y = wrap_any(s0 + i, H);
            lbuf[c * sr + i] = static_cast<Acc>(load_quadrant(im, q, x0 + c, y, img_w, img_h));
        }
    } else {  // working column = image row: contiguous along i
        for (int k = tid; k < cells; k += kThreads) {
            const int i = k % R, c = k / R;
            const int y = wrap_any(s0 + i, H);
            lbuf[c * sr + i] = static_cast<Acc>(load_quadrant(im, q, x0 + c, y, img_w, img_h));
        }
    }

    // Merge steps, deepest first: step k writes local depth nsteps-1-k.
    const int warp = tid >> 5, lane = tid & 31;
    for (int k = 0; k < nsteps; ++k) {
        __syncthreads();
        const Acc* src = ((nsteps - k) & 1) ? buf1 : buf0;
        Acc* dst = ((nsteps - 1 - k) & 1) ? buf1 : buf0;
        const int o_beg = soffs[k], o_end = soffs[k + 1];
        for (int o = o_beg + warp; o < o_end; o += kThreads / 32) {
            const int4 op = sops[o];
            const int r = op.w & 0xffff;
            const int rows = S + (op.w >> 16);
            const Acc* a = src + op.y * sr;
            Acc* d = dst + op.x * sr;
            if (op.z >= 0) {
                const Acc* b = src + op.z * sr + r;
                for (int i = lane; i < rows; i += 32) d[i] = a[i] + b[i];
            } else {
                for (int i = lane; i < rows; i += 32) d[i] = a[i];
            }
        }
    }
    __syncthreads();

    // Store the block root's S rows (values of local depth 0 live in buf0).
    const int rows_out = min(S, H - s0);
    if (!root_is_block) {
        Acc* __restrict__ dstw = ws + (size_t)slot * nbuf * W * ld;  // pass 0 output: buffer 0
        const int n = wb * rows_out;
        for (int k = tid; k < n; k += kThreads) {
            const int i = k % rows_out, c = k / rows_out;
            dstw[(size_t)(x0 + c) * ld + s0 + i] = buf0[c * sr + i];
        }
    } else {
        Out* o = reinterpret_cast<Out*>(out.ptr[q]) + (size_t)img_i * out.img_stride;
        const int n = wb * rows_out;
        if (out.layout == 0) {
            for (int k = tid; k < n; k += kThreads) {
                const int c = k % wb, i = k / wb;
                o[(size_t)(s0 + i) * W + c] = static_cast<Out>(buf0[c * sr + i]);
            }
        } else {
            for (int k = tid; k < n; k += kThreads) {
                const int i = k % rows_out, c = k / rows_out;
                o[(size_t)c * H + s0 + i] = static_cast<Out>(buf0[c * sr + i]);
            }
        }
    }
}

// ------------------------------------------------------------------- K2
// One fused upper pass.  grid: x = row tile (S rows), y = tile (G slopes of
// one band node), z = slot (image * nq + quadrant index).  A tile is a small
// program (plan.cpp build_tile): load the row windows of the frontier columns
// it depends on, run its merge ops level by level in shared memory (slot-
// major, row capacity L), then store its G columns -- into the other
// workspace buffer, or (root pass) straight into the output in the
// reference layout hough[s*W + t] (transform.cpp:80-83).
template <class Acc, class Out>
__global__ void __launch_bounds__(kThreads) k2_pass(PassDev ps, const Acc* __restrict__ src,
                                                     Acc* __restrict__ dst, long long slot_elems, int W, int H,
                                                     int ld, bool final_pass, OutDesc out, QuadSet qs, int img0) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* sm = reinterpret_cast<Acc*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kWarps = kThreads / 32;
    const PassTileDev tile = ps.tiles[blockIdx.y];
    const int S = ps.S, L = ps.L;
    const int s0 = blockIdx.x * S;
    const int slot = blockIdx.z;
    const Acc* __restrict__ in = src + (size_t)slot * slot_elems;

    // 1. windows of the input columns
    for (int l = warp; l < tile.load_cnt; l += kWarps) {
        const int4 ld4 = ps.loads[tile.load_beg + l];
        const Acc* __restrict__ col = in + (size_t)ld4.x * ld;
        Acc* __restrict__ d = sm + (size_t)ld4.y * L;
        const int n = S + ld4.w;
        int y = wrap_any(s0 + ld4.z + lane, H);
        for (int i = lane; i < n; i += 32) {
            d[i] = col[y];
            y += 32;
            if (y >= H) y = wrap_any(y, H);
        }
    }
    // 2. merge levels
    for (int k = 0; k < tile.nsteps; ++k) {
        __syncthreads();
        const int o_beg = ps.step_offs[tile.step_beg + k], o_end = ps.step_offs[tile.step_beg + k + 1];
        for (int o = o_beg + warp; o < o_end; o += kWarps) {
            const PassOpDev op = ps.ops[o];
            const Acc* a = sm + (size_t)op.a * L + op.ad;
            Acc* d = sm + (size_t)op.dst * L;
            const int n = S + op.ext;
            if (op.b >= 0) {
                const Acc* b = sm + (size_t)op.b * L + op.bd;
                for (int i = lane; i < n; i += 32) d[i] = a[i] + b[i];
            } else {
                for (int i = lane; i < n; i += 32) d[i] = a[i];
            }
        }
    }
    __syncthreads();
    // 3. store the tile's columns (window offset 0, rows [s0, s0 + S) clipped to H)
    const int rows = min(S, H - s0);
    if (!final_pass) {
        Acc* __restrict__ o = dst + (size_t)slot * slot_elems;
        for (int c = warp; c < tile.store_cnt; c += kWarps) {
            const int2 st = ps.stores[tile.store_beg + c];
            const Acc* sv = sm + (size_t)st.x * L;
            Acc* __restrict__ dcol = o + (size_t)st.y * ld + s0;
            for (int i = lane; i < rows; i += 32) dcol[i] = sv[i];
        }
    } else {
        const int nq = qs.n;
        Out* __restrict__ o =
            reinterpret_cast<Out*>(out.ptr[qs.code[slot % nq]]) + (size_t)(img0 + slot / nq) * out.img_stride;
        const int nc = tile.store_cnt;
        if (out.layout == 0) {
            // stores of a tile are consecutive slopes: write rows of nc contiguous t
            const int t0 = ps.stores[tile.store_beg].y;
            for (int k = tid; k < nc * rows; k += kThreads) {
                const int c = k % nc, i = k / nc;
                const int2 st = ps.stores[tile.store_beg + c];
                o[(size_t)(s0 + i) * W + t0 + c] = static_cast<Out>(sm[(size_t)st.x * L + i]);
            }
        } else {
            for (int c = warp; c < nc; c += kWarps) {
                const int2 st = ps.stores[tile.store_beg + c];
                const Acc* sv = sm + (size_t)st.x * L;
                Out* __restrict__ dcol = o + (size_t)st.y * H + s0;
                for (int i = lane; i < rows; i += 32) dcol[i] = static_cast<Out>(sv[i]);
            }
        }
    }
}

// --------------------------------------------------------------- absmax
template <class T>
__global__ void k_absmax(const T* __restrict__ in, long long n, unsigned long long* __restrict__ out) {
    unsigned long long m = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long v = static_cast<long long>(in[i]);
        const unsigned long long a = v < 0 ? 0ull - static_cast<unsigned long long>(v) : static_cast<unsigned long long>(v);
        m = a > m ? a : m;
    }
    for (int off = 16; off; off >>= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, m, off);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ------------------------------------------------------------ launchers
template <class In, class Acc, class Out>
int launch_typed(const GroupLaunch& g, cudaStream_t st, LaunchHook hook, void* ctx) {
    int launches = 0;
    const int nslots = g.nimg * g.qs.n;
    const size_t smem = k1_smem_bytes(g.acc_dtype, g.k1_max_width, g.k1_sr, g.k1_max_ops, g.k1_max_steps);
    auto k1 = k1_blocks<In, Acc, Out>;
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    Acc* ws = reinterpret_cast<Acc*>(g.ws);
    dim3 g1((g.H + g.S - 1) / g.S, g.nblocks, nslots);
    k1<<<g1, kThreads, smem, st>>>(reinterpret_cast<const In*>(g.img), g.img_w, g.img_h, g.img_stride, g.img0, g.qs,
                                   g.W, g.H, g.ld, g.S, g.blocks, g.shapes, g.step_offs, g.k1_ops, g.k1_max_width,
                                   g.k1_sr, g.k1_max_ops, ws, g.nbuf, g.root_is_block, g.out);
    ++launches;
    if (hook) hook(ctx, 1);
    if (g.root_is_block) return launches;
    const long long slot_elems = (long long)g.nbuf * g.W * g.ld;
    for (int p = 0; p < g.npasses; ++p) {
        const PassDev& ps = g.passes[p];
        const bool final_pass = (p == g.npasses - 1);
        const Acc* SRC = ws + (size_t)(p & 1) * g.W * g.ld;          // pass p reads buffer (p-1)%2 ... K1 wrote 0
        Acc* DST = ws + (size_t)((p + 1) & 1) * g.W * g.ld;
        const size_t smem2 = k2_smem_bytes(g.acc_dtype, ps.max_slots, ps.L);
        auto k2 = k2_pass<Acc, Out>;
        cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2));
        dim3 g2((g.H + ps.S - 1) / ps.S, ps.ntiles, nslots);
        k2<<<g2, kThreads, smem2, st>>>(ps, SRC, DST, slot_elems, g.W, g.H, g.ld, final_pass, g.out, g.qs, g.img0);
        ++launches;
        if (hook) hook(ctx, final_pass ? 3 : 2);
    }
    return launches;
}

}  // namespace

static size_t k1_ops_offset(int acc_dtype, int max_width, int sr) {
    const size_t esz = acc_dtype == kI64 ? 8 : 4;
    return (2 * static_cast<size_t>(max_width) * sr * esz + 15) / 16 * 16;
}

size_t k1_smem_bytes(int acc_dtype, int max_width, int sr, int max_ops, int max_steps) {
    return k1_ops_offset(acc_dtype, max_width, sr) + static_cast<size_t>(max_ops) * sizeof(int4) +
           static_cast<size_t>(max_steps + 1) * sizeof(int) + 16;
}

size_t k2_smem_bytes(int acc_dtype, int max_slots, int L) {
    const size_t esz = acc_dtype == kI64 ? 8 : 4;
    return static_cast<size_t>(max_slots) * L * esz;
}

int launch_group(const GroupLaunch& g, cudaStream_t st, LaunchHook hook, void* ctx) {
    const int in = g.in_dtype, acc = g.acc_dtype, out = g.out.dtype;
    if (acc == kI32 && out == kI32) {
        if (in == kU8) return launch_typed<uint8_t, int32_t, int32_t>(g, st, hook, ctx);
        if (in == kI32) return launch_typed<int32_t, int32_t, int32_t>(g, st, hook, ctx);
    }
    if (acc == kI32 && out == kI64) {
        if (in == kU8) return launch_typed<uint8_t, int32_t, long long>(g, st, hook, ctx);
        if (in == kI32) return launch_typed<int32_t, int32_t, long long>(g, st, hook, ctx);
        if (in == kI64) return launch_typed<long long, int32_t, long long>(g, st, hook, ctx);
    }
    if (acc == kI64 && out == kI64) {
        if (in == kU8) return launch_typed<uint8_t, long long, long long>(g, st, hook, ctx);
        if (in == kI32) return launch_typed<int32_t, long long, long long>(g, st, hook, ctx);
        if (in == kI64) return launch_typed<long long, long long, long long>(g, st, hook, ctx);
    }
    if (acc == kF32 && out == kF32) {
        if (in == kF32) return launch_typed<float, float, float>(g, st, hook, ctx);
        if (in == kU8) return launch_typed<uint8_t, float, float>(g, st, hook, ctx);
    }
    return -1;
}

void launch_absmax(const void* d_in, int dtype, long long n, unsigned long long* d_max, cudaStream_t st) {
    const int blocks = 148 * 4;
    if (dtype == kI32)
        k_absmax<int32_t><<<blocks, 256, 0, st>>>(reinterpret_cast<const int32_t*>(d_in), n, d_max);
    else if (dtype == kI64)
        k_absmax<long long><<<blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(d_in), n, d_max);
}

}  // namespace fhtb
