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

// ------------------------------------------------------------------- K1
// grid: x = row tile (S rows), y = block, z = slot (image * nq + quadrant idx)
template <class In, class Acc, class Out>
__global__ void __launch_bounds__(kThreads) k1_blocks(
    const In* __restrict__ img, int img_w, int img_h, long long img_stride, int img0, QuadSet qs, int W, int H,
    int ld, int S, const int4* __restrict__ blocks, const ShapeHdr* __restrict__ shapes,
    const int* __restrict__ step_offs, const int4* __restrict__ ops, int max_width, int sr, int max_ops,
    Acc* __restrict__ ws, bool root_is_block, OutDesc out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* buf0 = reinterpret_cast<Acc*>(smem_raw);
    Acc* buf1 = buf0 + (size_t)max_width * sr;
    int4* sops = reinterpret_cast<int4*>(buf1 + (size_t)max_width * sr);
    int* soffs = reinterpret_cast<int*>(sops + max_ops);

    const int tid = threadIdx.x;
    const int4 blk = blocks[blockIdx.y];
    const int x0 = blk.x, depth = blk.z;
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
        Acc* __restrict__ dstw = ws + (size_t)slot * 2 * W * ld + (size_t)(depth & 1) * W * ld;
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
// grid: x = op (output column), y = chunk of 4*kThreads rows, z = slot.
// src/dst are the two ping-pong buffers of the slot, or (to_out) the
// native-layout output.
template <class Acc, class Out, bool VEC>
__global__ void __launch_bounds__(kThreads) k2_level(const int4* __restrict__ ops, const Acc* __restrict__ src_buf,
                                                      Acc* __restrict__ dst_buf, long long slot_elems, int H, int ld,
                                                      bool to_out, OutDesc out, QuadSet qs, int img0) {
    const int4 op = ops[blockIdx.x];
    const int slot = blockIdx.z;
    const Acc* __restrict__ src = src_buf + (size_t)slot * slot_elems;
    const Acc* __restrict__ A = src + (size_t)op.y * ld;
    const Acc* __restrict__ B = src + (size_t)op.z * ld;
    const int r = op.w;
    const int s = (blockIdx.y * kThreads + threadIdx.x) * 4;
    if (s >= H) return;
    Out* __restrict__ D;
    if (!to_out) {
        D = reinterpret_cast<Out*>(dst_buf) + (size_t)slot * slot_elems + (size_t)op.x * ld;
    } else {
        const int nq = qs.n;
        D = reinterpret_cast<Out*>(out.ptr[qs.code[slot % nq]]) + (size_t)(img0 + slot / nq) * out.img_stride +
            (size_t)op.x * H;
    }
    Acc v[4];
    if (VEC && s + 3 < H) {
        if constexpr (sizeof(Acc) == 4) {
            const int4 a4 = *reinterpret_cast<const int4*>(A + s);
            v[0] = from_bits<Acc>(a4.x);
            v[1] = from_bits<Acc>(a4.y);
            v[2] = from_bits<Acc>(a4.z);
            v[3] = from_bits<Acc>(a4.w);
        } else {
            const longlong2 a0 = *reinterpret_cast<const longlong2*>(A + s);
            const longlong2 a1 = *reinterpret_cast<const longlong2*>(A + s + 2);
            v[0] = a0.x, v[1] = a0.y, v[2] = a1.x, v[3] = a1.y;
        }
        int j = wrap_once(s + r, H);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            v[e] = v[e] + B[j];
            j = wrap_once(j + 1, H);
        }
        if constexpr (VEC && std::is_same<Acc, Out>::value && sizeof(Acc) == 4) {
            if (!to_out) {
                *reinterpret_cast<int4*>(D + s) =
                    make_int4(to_bits(v[0]), to_bits(v[1]), to_bits(v[2]), to_bits(v[3]));
                return;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) D[s + e] = static_cast<Out>(v[e]);
    } else {
        int j = wrap_once(s + r, H);
        for (int e = 0; e < 4 && s + e < H; ++e) {
            D[s + e] = static_cast<Out>(A[s + e] + B[j]);
            j = wrap_once(j + 1, H);
        }
    }
}

// ------------------------------------------------------------------- K3
// Root level + transpose into hough[s*W + t].  grid: x = 32-slope tile,
// y = 32-shift tile, z = slot.  Block 32 x 8.
template <class Acc, class Out>
__global__ void __launch_bounds__(256) k3_root(const int4* __restrict__ ops, const Acc* __restrict__ ws, int W,
                                                int H, int ld, int src_par, OutDesc out, QuadSet qs, int img0) {
    __shared__ Acc tile[32][33];
    const int lane = threadIdx.x, ty = threadIdx.y;
    const int t0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
    const int slot = blockIdx.z;
    const Acc* __restrict__ src = ws + (size_t)slot * 2 * W * ld + (size_t)src_par * W * ld;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int tl = ty + 8 * j, t = t0 + tl, s = s0 + lane;
        if (t < W && s < H) {
            const int4 op = ops[t];
            const int jb = wrap_once(s + op.w, H);
            tile[tl][lane] = src[(size_t)op.y * ld + s] + src[(size_t)op.z * ld + jb];
        }
    }
    __syncthreads();
    const int nq = qs.n;
    Out* __restrict__ o =
        reinterpret_cast<Out*>(out.ptr[qs.code[slot % nq]]) + (size_t)(img0 + slot / nq) * out.img_stride;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int sl = ty + 8 * j, s = s0 + sl, t = t0 + lane;
        if (s < H && t < W) o[(size_t)s * W + t] = static_cast<Out>(tile[lane][sl]);
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
                                   g.k1_sr, g.k1_max_ops, ws, g.root_is_block, g.out);
    ++launches;
    if (hook) hook(ctx, 1);
    if (g.root_is_block) return launches;
    const bool vec = (g.ld % 4 == 0);
    for (int l = 0; l < g.nlevels; ++l) {
        const int d = g.level_depth[l];
        const int src_par = (d + 1) & 1, dst_par = d & 1;
        const long long slot_elems = 2LL * g.W * g.ld;
        const Acc* SRC = ws + (size_t)src_par * g.W * g.ld;
        Acc* DST = ws + (size_t)dst_par * g.W * g.ld;
        if (d > 0 || g.out.layout == 1) {
            const bool to_out = (d == 0);
            dim3 g2(g.level_nops[l], (g.H + 4 * kThreads - 1) / (4 * kThreads), nslots);
            if (!to_out) {
                if (vec)
                    k2_level<Acc, Acc, true><<<g2, kThreads, 0, st>>>(g.level_ops[l], SRC, DST, slot_elems, g.H, g.ld,
                                                                     false, g.out, g.qs, g.img0);
                else
                    k2_level<Acc, Acc, false><<<g2, kThreads, 0, st>>>(g.level_ops[l], SRC, DST, slot_elems, g.H, g.ld,
                                                                      false, g.out, g.qs, g.img0);
            } else {
                if (vec)
                    k2_level<Acc, Out, true><<<g2, kThreads, 0, st>>>(g.level_ops[l], SRC, DST, slot_elems, g.H, g.ld,
                                                                     true, g.out, g.qs, g.img0);
                else
                    k2_level<Acc, Out, false><<<g2, kThreads, 0, st>>>(g.level_ops[l], SRC, DST, slot_elems, g.H, g.ld,
                                                                      true, g.out, g.qs, g.img0);
            }
        } else {
            dim3 g3((g.W + 31) / 32, (g.H + 31) / 32, nslots);
            k3_root<Acc, Out><<<g3, dim3(32, 8), 0, st>>>(g.level_ops[l], ws, g.W, g.H, g.ld, src_par, g.out, g.qs,
                                                          g.img0);
        }
        ++launches;
        if (hook) hook(ctx, (d > 0 || g.out.layout == 1) ? 2 : 3);
    }
    return launches;
}

}  // namespace

size_t k1_smem_bytes(int acc_dtype, int max_width, int sr, int max_ops, int max_steps) {
    const size_t esz = acc_dtype == kI64 ? 8 : 4;
    return 2 * static_cast<size_t>(max_width) * sr * esz + static_cast<size_t>(max_ops) * sizeof(int4) +
           static_cast<size_t>(max_steps + 1) * sizeof(int) + 16;
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
