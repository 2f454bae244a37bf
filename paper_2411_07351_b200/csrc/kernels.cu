// kernels.cu -- sm_100a kernels for the FHT2D merge DP (transform.cpp:35-58).
//
// Pass 0 (blocks: maximal subtrees of width <= 32), loading the input tile in
// the quadrant's orientation straight from the row-major image (no flip /
// transpose copies, quadrants.cpp:7-21):
//   k1_by32      K1P: width-32 Brady-Yong blocks, op indices computed
//                arithmetically, levels 1-2 in registers, 3-5 in shared memory.
//   k1_blocks    K1: any other block shape, table-driven ops.
// Passes 1.. (the tree above the blocks in bands of <= 4 levels):
//   k2_pass      K2: one tile program per CTA (cp.async windows of the
//                frontier columns, merge ops level by level in shared memory);
//                the last band stores the root in the reference layout
//                hough[s*W + t] (transform.cpp:80-83), optionally widened.
// Plus k_merge_root (the multi-GPU root split) and k_absmax (overflow budget).
// The path is a gather-add: no contraction, so no tensor cores.  Each level
// costs a shared-memory round trip per cell, so the kernels are bound by the
// shared-memory/LSU pipe at this design point; see DESIGN.md §4.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>
#include <type_traits>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"

namespace fhtb {

namespace {

constexpr int kThreads = 512;

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ int wrap_any(int j, int H) {
    if (j >= H) j -= H;
    if (j >= H) j %= H;
    return j;
}

constexpr int kU = 8;  // independent global loads in flight per lane

// d[i] = col[(start + i) mod H] for i in [0, n), one warp, kU loads in flight per lane.
template <class Acc, class Src>
__device__ __forceinline__ void warp_load_window(Acc* __restrict__ d, const Src* __restrict__ col, int start, int n,
                                                 int H, int lane) {
    if (start + n <= H) {  // no wrap: plain contiguous run
        for (int i0 = 0; i0 < n; i0 += 32 * kU) {
            Src v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < n) v[u] = col[start + i];
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < n) d[i] = static_cast<Acc>(v[u]);
            }
        }
        return;
    }
    for (int i0 = 0; i0 < n; i0 += 32 * kU) {
        Src v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = i0 + u * 32 + lane;
            if (i < n) v[u] = col[wrap_any(start + i, H)];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = i0 + u * 32 + lane;
            if (i < n) d[i] = static_cast<Acc>(v[u]);
        }
    }
}

// Shared-memory merge of one column window: d[i] = a[i] + b[i] (b null: copy).
template <class Acc>
__device__ __forceinline__ void warp_merge(Acc* d, const Acc* a, const Acc* b, int n, int lane) {
    constexpr int U = 4;
    if (b) {
        for (int i0 = 0; i0 < n; i0 += 32 * U) {
            Acc x[U], y[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < n) x[u] = a[i], y[u] = b[i];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < n) d[i] = x[u] + y[u];
            }
        }
    } else {
        for (int i = lane; i < n; i += 32) d[i] = a[i];
    }
}

// Select from the by-value parameter structs without dynamic indexing (which
// would copy them to local memory).
__device__ __forceinline__ int quad_code(const QuadSet& qs, int i) {
    return i == 0 ? qs.code[0] : i == 1 ? qs.code[1] : i == 2 ? qs.code[2] : qs.code[3];
}
// slot = image * nq + quadrant index, nq in 1..4, without a runtime division
__device__ __forceinline__ void split_slot(int slot, int nq, int& img, int& qi) {
    if (nq == 4) img = slot >> 2, qi = slot & 3;
    else if (nq == 2) img = slot >> 1, qi = slot & 1;
    else if (nq == 1) img = slot, qi = 0;
    else img = slot / 3, qi = slot - 3 * img;  // constant divisor
}
__device__ __forceinline__ void* out_ptr(const OutDesc& o, int q) {
    return q == 0 ? o.ptr[0] : q == 1 ? o.ptr[1] : q == 2 ? o.ptr[2] : o.ptr[3];
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

__device__ __forceinline__ int4 lds4(const void* p) { return *reinterpret_cast<const int4*>(p); }
__device__ __forceinline__ void sts4(void* p, int4 v) { *reinterpret_cast<int4*>(p) = v; }

// 32-bit shared-window addressing for the merge inner loops (keeps the
// compiler from rematerialising the shared window base per access).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ int4 lds4u(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts4u(uint32_t a, int4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// d[k] = a[k] + b[k + M] for one lane's 4 rows; b0/b1 are the aligned b
// vectors at and after the lane's rows.
template <int M, class Acc>
__device__ __forceinline__ int4 add_shift(int4 av, int4 b0, int4 b1) {
    const int bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    return make_int4(to_bits<Acc>(from_bits<Acc>(av.x) + from_bits<Acc>(bv[M + 0])),
                     to_bits<Acc>(from_bits<Acc>(av.y) + from_bits<Acc>(bv[M + 1])),
                     to_bits<Acc>(from_bits<Acc>(av.z) + from_bits<Acc>(bv[M + 2])),
                     to_bits<Acc>(from_bits<Acc>(av.w) + from_bits<Acc>(bv[M + 3])));
}

// One op, one warp, 4-byte types: rows [0, n) of d = a + (b shifted by M),
// byte addresses in the shared window (d, a, bb 16-byte aligned, bb the
// aligned base of the shifted b).  Lanes own 4 consecutive rows, lanes
// contiguous (conflict-free); warp-uniform full 128-row chunks two at a time
// (all loads before the adds), then one predicated tail chunk.
template <int M, class Acc>
__device__ __forceinline__ void rows_op(uint32_t d, uint32_t a, uint32_t bb, int n, int lane) {
    const int nfull = n >> 7;
    uint32_t off = lane * 16u;
    int c = 0;
    for (; c + 2 <= nfull; c += 2, off += 1024u) {
        const int4 a0 = lds4u(a + off), a1 = lds4u(a + off + 512u);
        const int4 p0 = lds4u(bb + off), p1 = lds4u(bb + off + 512u);
        int4 q0 = p0, q1 = p1;
        if (M) {
            q0 = lds4u(bb + off + 16u);
            q1 = lds4u(bb + off + 528u);
        }
        sts4u(d + off, add_shift<M, Acc>(a0, p0, q0));
        sts4u(d + off + 512u, add_shift<M, Acc>(a1, p1, q1));
    }
    if (c < nfull) {
        const int4 a0 = lds4u(a + off), p0 = lds4u(bb + off);
        const int4 q0 = M ? lds4u(bb + off + 16u) : p0;
        sts4u(d + off, add_shift<M, Acc>(a0, p0, q0));
        off += 512u;
    }
    if (lane * 4 < n - (nfull << 7)) {
        const int4 a0 = lds4u(a + off), p0 = lds4u(bb + off);
        const int4 q0 = M ? lds4u(bb + off + 16u) : p0;
        sts4u(d + off, add_shift<M, Acc>(a0, p0, q0));
    }
}

// TMA windows in k2_pass: the residue (in bytes) of window w, two bits per
// window in two 64-bit masks
__device__ __forceinline__ uint32_t win_adj(unsigned long long m0, unsigned long long m1, unsigned w) {
    const unsigned long long m = (w & 32) ? m1 : m0;
    return static_cast<uint32_t>((m >> (2 * (w & 31))) & 3ull) << 2;
}

__device__ __forceinline__ int lds1u(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts1u(uint32_t a, int v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// An address the compiler must treat as opaque: the inner loops add only
// compile-time offsets to it, which ptxas folds into the LDS/STS immediate.
// (Otherwise NVVM rewrites t[k] + lane*4 + c as t[k] + (lane*4 | c) to share
// the OR across terms -- one extra IADD per shared load.)
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm("" : "+r"(x));
    return x;
}
template <class Acc>
__device__ __forceinline__ int add_bits(int x, int y) {
    return to_bits<Acc>(from_bits<Acc>(x) + from_bits<Acc>(y));
}

// u16 pair mode: a 32-bit word j of a working column holds
// rows j (low half) and j + D (high half), both < 2^16 (a node of width w
// sums w u8 leaves: w * 255 < 2^16 for every node below the root when the
// root's children are at most 257 wide).  One integer add then advances
// both rows, and the shifts of the DP -- the same for every row -- act on
// whole words.  pack_pair_u8x4: 4 staged leaf rows of each half -> 4 words.
__device__ __forceinline__ int4 pack_pair_u8x4(uint32_t lo, uint32_t hi) {
    const uint32_t t0 = __byte_perm(lo, hi, 0x5410), t1 = __byte_perm(lo, hi, 0x7632);  // lo0 lo1 hi0 hi1 | ..
    return make_int4(static_cast<int>(__byte_perm(t0, 0u, 0x4240)), static_cast<int>(__byte_perm(t0, 0u, 0x4341)),
                     static_cast<int>(__byte_perm(t1, 0u, 0x4240)), static_cast<int>(__byte_perm(t1, 0u, 0x4341)));
}

// Word j of the pair layout for j in [D, H): rows j and (j + D) mod H =
// j - D + e (e = 2D - H), i.e. the high half of word j - D and the low half
// of word j - D + e.  The tile computes words [0, D) only (every row once).
__device__ __forceinline__ int pair_extra_word(int w_k, int w_ke) { return static_cast<int>(__byte_perm(w_k, w_ke, 0x5432)); }

// The same op with rows interleaved over lanes (lane l owns rows l, l+32,
// ...): 32 consecutive words are conflict-free at any alignment, so the
// shifted operand costs one wavefront per 32 rows like the aligned ones
// (the 4-rows-per-lane form needs a second, 4-way conflicted, b load when
// the shift is not a multiple of 4).  b is the exact (unaligned) address.
template <class Acc>
__device__ __forceinline__ void rows_op_s(uint32_t d, uint32_t a, uint32_t b, int n, int lane) {
    constexpr int U = 4;  // 128 rows per step (8 measured slower: code size)
    const uint32_t lo = lane * 4u;
    int i0 = 0;
    for (; i0 + 32 * U <= n; i0 += 32 * U) {
        int x[U], y[U];
        const uint32_t o = lo + i0 * 4u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x[u] = lds1u(a + o + 128u * u);
            y[u] = lds1u(b + o + 128u * u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) sts1u(d + o + 128u * u, add_bits<Acc>(x[u], y[u]));
    }
    for (; i0 < n; i0 += 32)
        if (i0 + lane < n) {
            const uint32_t o = lo + i0 * 4u;
            sts1u(d + o, add_bits<Acc>(lds1u(a + o), lds1u(b + o)));
        }
}

// A level-pair op (plan.hpp PassOpN): d[i] = sum of K shifted windows,
// added in the tree's order -- (first child's terms) + (second child's).
template <class Acc, int K, int SPLIT>
__device__ __forceinline__ int sum_terms(const int (&v)[4]) {
    if constexpr (K == 2) return add_bits<Acc>(v[0], v[1]);
    if constexpr (K == 3 && SPLIT == 2) return add_bits<Acc>(add_bits<Acc>(v[0], v[1]), v[2]);
    if constexpr (K == 3) return add_bits<Acc>(v[0], add_bits<Acc>(v[1], v[2]));
    return add_bits<Acc>(add_bits<Acc>(v[0], v[1]), add_bits<Acc>(v[2], v[3]));
}
template <class Acc, int K, int SPLIT>
__device__ __forceinline__ void rows_op_terms(uint32_t d, const uint32_t (&t)[4], int n, int lane) {
    constexpr int U = 4;
    const uint32_t lo = lane * 4u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
    const uint32_t dd = opaque(d + lo);
    int i0 = 0;
    for (; i0 + 32 * U <= n; i0 += 32 * U) {
        int v[U][4];
        const uint32_t o = i0 * 4u;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) v[u][k] = lds1u(p[k] + o + 128u * u);
#pragma unroll
        for (int u = 0; u < U; ++u) sts1u(dd + o + 128u * u, sum_terms<Acc, K, SPLIT>(v[u]));
    }
    for (; i0 < n; i0 += 32)
        if (i0 + lane < n) {
            const uint32_t o = i0 * 4u;
            int v[4];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = lds1u(p[k] + o);
            sts1u(dd + o, sum_terms<Acc, K, SPLIT>(v));
        }
}

// A stored column of a non-root band written straight to the workspace
// from registers (lane = row: 128 contiguous bytes per warp store).
template <class Acc, int K, int SPLIT>
__device__ __forceinline__ void rows_op_terms_global(Acc* __restrict__ g, const uint32_t (&t)[4], int n, int lane) {
    constexpr int U = 4;
    const uint32_t lo = lane * 4u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
    int i0 = 0;
    for (; i0 + 32 * U <= n; i0 += 32 * U) {
        int v[U][4];
        const uint32_t o = i0 * 4u;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) v[u][k] = lds1u(p[k] + o + 128u * u);
#pragma unroll
        for (int u = 0; u < U; ++u) g[i0 + 32 * u + lane] = from_bits<Acc>(sum_terms<Acc, K, SPLIT>(v[u]));
    }
    for (; i0 < n; i0 += 32)
        if (i0 + lane < n) {
            const uint32_t o = i0 * 4u;
            int v[4];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = lds1u(p[k] + o);
            g[i0 + lane] = from_bits<Acc>(sum_terms<Acc, K, SPLIT>(v));
        }
}

// rows_op_terms for 256 <= n < 288 (a full 256-row tile plus a halo of < 32
// rows): 8 whole groups with compile-time offsets, then one lane-predicated
// group -- no loop control.
// (NH = 2: 256 <= n < 288; NH = 1: the same for 128-row tiles, 128 <= n < 160)
template <class Acc, int K, int SPLIT, int NH = 2>
__device__ __forceinline__ void rows_op_terms_256(uint32_t d, const uint32_t (&t)[4], int n, int lane) {
    const uint32_t lo = lane * 4u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
    const uint32_t dd = opaque(d + lo);
#pragma unroll
    for (int half = 0; half < NH; ++half) {
        int v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) v[u][k] = lds1u(p[k] + 512u * half + 128u * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) sts1u(dd + 512u * half + 128u * u, sum_terms<Acc, K, SPLIT>(v[u]));
    }
    if (128 * NH + lane < n) {
        int v[4];
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = lds1u(p[k] + 512u * NH);
        sts1u(dd + 512u * NH, sum_terms<Acc, K, SPLIT>(v));
    }
}

// rows_op_terms_global for exactly 256 rows (a full tile): no loop control
template <class Acc, int K, int SPLIT, int NH = 2>
__device__ __forceinline__ void rows_op_terms_global_256(Acc* __restrict__ g, const uint32_t (&t)[4], int lane) {
    const uint32_t lo = lane * 4u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
#pragma unroll
    for (int half = 0; half < NH; ++half) {
        int v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) v[u][k] = lds1u(p[k] + 512u * half + 128u * u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            g[128 * half + 32 * u + lane] = from_bits<Acc>(sum_terms<Acc, K, SPLIT>(v[u]));
    }
}

// The root step of the u16 pair mode: the children's sums x (first child)
// and y (second child) are packed words (each half < 2^16); the root adds
// them half by half into two 32-bit columns -- rows [0, S) of the tile to d,
// rows [D, D + S) to dh.  Same add order as the tree (x + y per row).
template <int K, int SPLIT>
__device__ __forceinline__ void child_sums(const int (&v)[4], uint32_t& x, uint32_t& y) {
    const uint32_t a = static_cast<uint32_t>(v[0]), b = static_cast<uint32_t>(v[1]), c = static_cast<uint32_t>(v[2]),
                   d = static_cast<uint32_t>(v[3]);
    if constexpr (K == 1) x = a, y = 0u;
    else if constexpr (K == 2) x = a, y = b;
    else if constexpr (K == 3 && SPLIT == 2) x = a + b, y = c;
    else if constexpr (K == 3) x = a, y = b + c;
    else x = a + b, y = c + d;
}
template <int K, int SPLIT>
__device__ __forceinline__ void rows_op_widen(uint32_t d, uint32_t dh, const uint32_t (&t)[4], int n, int lane) {
    constexpr int U = 2;
    const uint32_t lo = lane * 4u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
    const uint32_t dd = opaque(d + lo), ddh = opaque(dh + lo);
    for (int i0 = 0; i0 < n; i0 += 32 * U) {
        int v[U][4];
        const uint32_t o = i0 * 4u;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + 32 * u + lane < n)
#pragma unroll
                for (int k = 0; k < K; ++k) v[u][k] = lds1u(p[k] + o + 128u * u);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + 32 * u + lane < n) {
                uint32_t x, y;
                child_sums<K, SPLIT>(v[u], x, y);
                sts1u(dd + o + 128u * u, static_cast<int>((x & 0xffffu) + (y & 0xffffu)));
                sts1u(ddh + o + 128u * u, static_cast<int>((x >> 16) + (y >> 16)));
            }
    }
}
// rows_op_widen for exactly 256 words (a full pair-mode tile, the root has
// no halo): 8 whole row groups with compile-time offsets, no predicates.
template <int K, int SPLIT>
__device__ __forceinline__ void rows_op_widen_256(uint32_t d, uint32_t dh, const uint32_t (&t)[4], int lane) {
    const uint32_t lo = lane * 4u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
    const uint32_t dd = opaque(d + lo), ddh = opaque(dh + lo);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int v[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) v[u][k] = lds1u(p[k] + 256u * q + 128u * u);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            uint32_t x, y;
            child_sums<K, SPLIT>(v[u], x, y);
            sts1u(dd + 256u * q + 128u * u, static_cast<int>((x & 0xffffu) + (y & 0xffffu)));
            sts1u(ddh + 256u * q + 128u * u, static_cast<int>((x >> 16) + (y >> 16)));
        }
    }
}

// 8-byte accumulators (int64): the same level-pair ops on 64-bit words --
// lane l owns rows l, l + 32, ... (256 bytes per 32 rows, two wavefronts).
__device__ __forceinline__ long long lds2u(uint32_t a) {
    long long v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts2u(uint32_t a, long long v) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
template <int K, int SPLIT>
__device__ __forceinline__ long long sum_terms64(const long long (&v)[4]) {
    if constexpr (K == 2) return v[0] + v[1];
    if constexpr (K == 3 && SPLIT == 2) return (v[0] + v[1]) + v[2];
    if constexpr (K == 3) return v[0] + (v[1] + v[2]);
    return (v[0] + v[1]) + (v[2] + v[3]);
}
// d (shared) or g (global, DIRECT) = the op's K shifted windows, rows [0, n)
template <int K, int SPLIT, bool GLOBAL>
__device__ __forceinline__ void rows_op_terms64(uint32_t d, long long* __restrict__ g, const uint32_t (&t)[4], int n,
                                                int lane) {
    constexpr int U = 4;
    const uint32_t lo = lane * 8u;
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = opaque(t[k] + lo);
    const uint32_t dd = opaque(d + lo);
    int i0 = 0;
    for (; i0 + 32 * U <= n; i0 += 32 * U) {
        long long v[U][4];
        const uint32_t o = i0 * 8u;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) v[u][k] = lds2u(p[k] + o + 256u * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long r = sum_terms64<K, SPLIT>(v[u]);
            if constexpr (GLOBAL) g[i0 + 32 * u + lane] = r;
            else sts2u(dd + o + 256u * u, r);
        }
    }
    for (; i0 < n; i0 += 32)
        if (i0 + lane < n) {
            const uint32_t o = i0 * 8u;
            long long v[4];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = lds2u(p[k] + o);
            const long long r = sum_terms64<K, SPLIT>(v);
            if constexpr (GLOBAL) g[i0 + lane] = r;
            else sts2u(dd + o, r);
        }
}
template <int NWARPS, bool DIRECT>
__device__ __forceinline__ void run_step_terms64(uint32_t base, const int4* __restrict__ ops, int o_beg, int o_end,
                                                 int warp, int lane, long long* __restrict__ gdst = nullptr, int ld = 0,
                                                 int rows_out = 0) {
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const int4 h = ops[2 * o], q = ops[2 * o + 1];
        const uint32_t d = base + static_cast<uint32_t>(h.x);
        const uint32_t t[4] = {base + static_cast<uint32_t>(h.w), base + static_cast<uint32_t>(q.x),
                               base + static_cast<uint32_t>(q.y), base + static_cast<uint32_t>(q.z)};
        const int nt = h.z & 7, gc = (h.z >> 3) - 1, sp2 = (q.w & 15) == 2;
        long long* __restrict__ g = DIRECT && gdst != nullptr && gc >= 0 ? gdst + (size_t)gc * ld : nullptr;
        const int n = g ? rows_out : h.y;
        if (g) {  // a stored column (non-root band): straight to the workspace
            if (nt == 4) rows_op_terms64<4, 2, true>(0u, g, t, n, lane);
            else if (nt == 2) rows_op_terms64<2, 1, true>(0u, g, t, n, lane);
            else if (nt == 3 && sp2) rows_op_terms64<3, 2, true>(0u, g, t, n, lane);
            else if (nt == 3) rows_op_terms64<3, 1, true>(0u, g, t, n, lane);
            else
                for (int i = lane; i < n; i += 32) g[i] = lds2u(t[0] + 8u * i);
            continue;
        }
        if (nt == 4) rows_op_terms64<4, 2, false>(d, nullptr, t, n, lane);
        else if (nt == 2) rows_op_terms64<2, 1, false>(d, nullptr, t, n, lane);
        else if (nt == 3 && sp2) rows_op_terms64<3, 2, false>(d, nullptr, t, n, lane);
        else if (nt == 3) rows_op_terms64<3, 1, false>(d, nullptr, t, n, lane);
        else
            for (int i = lane; i < n; i += 32) sts2u(d + 8u * i, lds2u(t[0] + 8u * i));
    }
}

template <int NWARPS>
__device__ __forceinline__ void run_step_widen(uint32_t base, const int4* __restrict__ ops, int o_beg, int o_end,
                                               int warp, int lane) {
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const int4 h = ops[2 * o], q = ops[2 * o + 1];
        const uint32_t d = base + static_cast<uint32_t>(h.x), dh = base + (static_cast<uint32_t>(q.w) >> 4);
        const uint32_t t[4] = {base + static_cast<uint32_t>(h.w), base + static_cast<uint32_t>(q.x),
                               base + static_cast<uint32_t>(q.y), base + static_cast<uint32_t>(q.z)};
        const int n = h.y, nt = h.z & 7, split = q.w & 15;
        if (nt == 4 && n == 256) rows_op_widen_256<4, 2>(d, dh, t, lane);
        else if (nt == 4) rows_op_widen<4, 2>(d, dh, t, n, lane);
        else if (nt == 2) rows_op_widen<2, 1>(d, dh, t, n, lane);
        else if (nt == 3 && split == 2) rows_op_widen<3, 2>(d, dh, t, n, lane);
        else if (nt == 3) rows_op_widen<3, 1>(d, dh, t, n, lane);
        else rows_op_widen<1, 1>(d, dh, t, n, lane);
    }
}

// The level-pair step and root step of the pair-mode root band (k2_pair_pipe)
// with the op records addressed as shared-window offsets: the records are
// read with ld.shared at a 32-bit address, so no op re-derives the shared
// window base from a generic pointer (10 uniform instructions per op).
template <int NWARPS>
__device__ __forceinline__ void run_step_terms_s(uint32_t base, uint32_t ops, int o_beg, int o_end, int warp, int lane) {
    using Acc = int;
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const int4 h = lds4u(ops + 32u * o), q = lds4u(ops + 32u * o + 16u);
        const uint32_t d = base + static_cast<uint32_t>(h.x);
        const uint32_t t[4] = {base + static_cast<uint32_t>(h.w), base + static_cast<uint32_t>(q.x),
                               base + static_cast<uint32_t>(q.y), base + static_cast<uint32_t>(q.z)};
        const int n = h.y, nt = h.z & 7;
        if (nt == 4) {
            if (n >= 256 && n < 288) rows_op_terms_256<Acc, 4, 2>(d, t, n, lane);
            else rows_op_terms<Acc, 4, 2>(d, t, n, lane);
        } else if (nt == 2) {
            if (n >= 256 && n < 288) rows_op_terms_256<Acc, 2, 1>(d, t, n, lane);
            else rows_op_terms<Acc, 2, 1>(d, t, n, lane);
        } else if (nt == 3) {
            if ((q.w & 15) == 2) rows_op_terms<Acc, 3, 2>(d, t, n, lane);
            else rows_op_terms<Acc, 3, 1>(d, t, n, lane);
        } else {
            for (int i = lane; i < n; i += 32) sts1u(d + 4u * i, lds1u(t[0] + 4u * i));
        }
    }
}
template <int NWARPS>
__device__ __forceinline__ void run_step_widen_s(uint32_t base, uint32_t ops, int o_beg, int o_end, int warp, int lane) {
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const int4 h = lds4u(ops + 32u * o), q = lds4u(ops + 32u * o + 16u);
        const uint32_t d = base + static_cast<uint32_t>(h.x), dh = base + (static_cast<uint32_t>(q.w) >> 4);
        const uint32_t t[4] = {base + static_cast<uint32_t>(h.w), base + static_cast<uint32_t>(q.x),
                               base + static_cast<uint32_t>(q.y), base + static_cast<uint32_t>(q.z)};
        const int n = h.y, nt = h.z & 7, split = q.w & 15;
        if (nt == 4 && n == 256) rows_op_widen_256<4, 2>(d, dh, t, lane);
        else if (nt == 4) rows_op_widen<4, 2>(d, dh, t, n, lane);
        else if (nt == 2) rows_op_widen<2, 1>(d, dh, t, n, lane);
        else if (nt == 3 && split == 2) rows_op_widen<3, 2>(d, dh, t, n, lane);
        else if (nt == 3) rows_op_widen<3, 1>(d, dh, t, n, lane);
        else rows_op_widen<1, 1>(d, dh, t, n, lane);
    }
}

template <class Acc, int NWARPS, bool DIRECT, bool WADJ = false>
__device__ __forceinline__ void run_step_terms(uint32_t base, const int4* __restrict__ ops, int o_beg, int o_end,
                                               int warp, int lane, Acc* __restrict__ gdst = nullptr, int ld = 0,
                                               int rows_out = 0, const int* __restrict__ wsl = nullptr,
                                               unsigned long long m0 = 0, unsigned long long m1 = 0) {
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const int4 h = ops[2 * o], q = ops[2 * o + 1];
        const uint32_t d = base + static_cast<uint32_t>(h.x);
        uint32_t t[4] = {base + static_cast<uint32_t>(h.w), base + static_cast<uint32_t>(q.x),
                         base + static_cast<uint32_t>(q.y), base + static_cast<uint32_t>(q.z)};
        if constexpr (WADJ) {  // terms reading a TMA window: + its alignment residue
            const unsigned ws = static_cast<unsigned>(wsl[o]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned w = (ws >> (8 * k)) & 0xffu;
                if (w != 0xffu) t[k] += win_adj(m0, m1, w);
            }
        }
        const int n = h.y, nt = h.z & 7, gc = (h.z >> 3) - 1;
        if (DIRECT && gdst != nullptr && gc >= 0) {  // a stored column (non-root band): straight to the workspace
            Acc* __restrict__ g = gdst + (size_t)gc * ld;
            if (nt == 4 && rows_out == 256) rows_op_terms_global_256<Acc, 4, 2>(g, t, lane);
            else if (nt == 4 && rows_out == 128) rows_op_terms_global_256<Acc, 4, 2, 1>(g, t, lane);
            else if (nt == 4) rows_op_terms_global<Acc, 4, 2>(g, t, rows_out, lane);
            else if (nt == 2 && rows_out == 256) rows_op_terms_global_256<Acc, 2, 1>(g, t, lane);
            else if (nt == 2) rows_op_terms_global<Acc, 2, 1>(g, t, rows_out, lane);
            else if (nt == 3 && (q.w & 15) == 2) rows_op_terms_global<Acc, 3, 2>(g, t, rows_out, lane);
            else if (nt == 3) rows_op_terms_global<Acc, 3, 1>(g, t, rows_out, lane);
            else
                for (int i = lane; i < rows_out; i += 32) g[i] = from_bits<Acc>(lds1u(t[0] + 4u * i));
            continue;
        }
        if (nt == 4) {
            if (n >= 256 && n < 288) rows_op_terms_256<Acc, 4, 2>(d, t, n, lane);
            else if (n >= 128 && n < 160) rows_op_terms_256<Acc, 4, 2, 1>(d, t, n, lane);
            else rows_op_terms<Acc, 4, 2>(d, t, n, lane);
        } else if (nt == 2) {
            if (n >= 256 && n < 288) rows_op_terms_256<Acc, 2, 1>(d, t, n, lane);
            else rows_op_terms<Acc, 2, 1>(d, t, n, lane);
        } else if (nt == 3) {
            if ((q.w & 15) == 2) rows_op_terms<Acc, 3, 2>(d, t, n, lane);
            else rows_op_terms<Acc, 3, 1>(d, t, n, lane);
        } else {  // a single term: copy
            for (int i = lane; i < n; i += 32) sts1u(d + 4u * i, lds1u(t[0] + 4u * i));
        }
    }
}

// K2 window load, 4-byte types: d[i] = col[(start + i) mod H], i < n, with
// d 16-byte aligned.  The run up to the wrap point is copied with 16-byte
// loads/stores when `start` is 4-aligned (columns are: ld % 4 == 0); the
// rest (after the wrap) with unrolled scalar loads.
template <class Acc>
__device__ __forceinline__ void warp_load_window_v(Acc* __restrict__ d, const Acc* __restrict__ col, int start,
                                                   int n, int H, int lane) {
    int done = 0;
    if constexpr (sizeof(Acc) == 4) {
        if ((start & 3) == 0) {
            const int run = min(n, H - start) & ~3;
            const int4* __restrict__ src = reinterpret_cast<const int4*>(col + start);
            for (int k0 = 0; k0 < run / 4; k0 += 32 * 2) {
                int4 v[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int k = k0 + u * 32 + lane;
                    if (k < run / 4) v[u] = src[k];
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int k = k0 + u * 32 + lane;
                    if (k < run / 4) sts4(d + 4 * k, v[u]);
                }
            }
            done = run;
        }
    }
    if (done < n) warp_load_window(d + done, col, wrap_any(start + done, H), n - done, H, lane);
}

// One merge step of a tile program, all warps of the CTA, warp per op:
//   sm[dst*stride + i] = sm[a*stride + ad + i] + sm[b*stride + bd + i],
//   i < S + ext (b < 0: copy).
// a and dst are 16-byte aligned (ad % 4 == 0); b is read from its aligned
// base and the warp-uniform residue bd & 3 selects a specialised loop.
template <class Acc, int NWARPS>
__device__ __forceinline__ void run_step(Acc* sm, int stride, const PassOpDev* __restrict__ ops, int o_beg,
                                         int o_end, int S, int warp, int lane) {
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const PassOpDev op = ops[o];
        warp_merge(sm + (size_t)op.dst * stride, sm + (size_t)op.a * stride + op.ad,
                   op.b >= 0 ? sm + (size_t)op.b * stride + op.bd : nullptr, S + op.ext, lane);
    }
}

// 4-byte path with ops baked on the host into 16-byte records of shared
// byte offsets: {dst, a (+ad), b aligned base | (bd & 3)  (-1: copy), rows}.
template <class Acc, int NWARPS, bool SC = false>
__device__ __forceinline__ void run_step_baked(uint32_t base, const int4* __restrict__ ops, int o_beg, int o_end,
                                               int warp, int lane) {
    for (int o = o_beg + warp; o < o_end; o += NWARPS) {
        const int4 op = ops[o];
        const uint32_t d = base + static_cast<uint32_t>(op.x), a = base + static_cast<uint32_t>(op.y);
        const int n = op.w;
        if (op.z < 0) {
            for (int i = lane * 4; i < n; i += 128) sts4u(d + i * 4u, lds4u(a + i * 4u));
            continue;
        }
        const uint32_t bb = base + static_cast<uint32_t>(op.z & ~15);
        if (SC) {
            const uint32_t b = bb + 4u * static_cast<uint32_t>(op.z & 3);
            if (n >= 256 && n < 288) {  // a full tile plus a short halo: fixed shape
                const uint32_t t[4] = {a, b, 0u, 0u};
                rows_op_terms_256<Acc, 2, 1>(d, t, n, lane);
            } else {
                rows_op_s<Acc>(d, a, b, n, lane);
            }
            continue;
        }
        switch (op.z & 3) {
            case 0: rows_op<0, Acc>(d, a, bb, n, lane); break;
            case 1: rows_op<1, Acc>(d, a, bb, n, lane); break;
            case 2: rows_op<2, Acc>(d, a, bb, n, lane); break;
            default: rows_op<3, Acc>(d, a, bb, n, lane); break;
        }
    }
}

// Column store smem -> global, rows [0, n): 16-byte stores when the global
// column start is 16-byte aligned (4-byte types), scalar tail.
template <class Acc, class Out>
__device__ __forceinline__ void warp_store_col(Out* __restrict__ g, const Acc* s, int n, bool aligned, int lane) {
    int done = 0;
    if constexpr (sizeof(Acc) == 4 && std::is_same<Acc, Out>::value) {
        if (aligned) {
            const int n4 = n & ~3;
            for (int i = lane * 4; i < n4; i += 128) *reinterpret_cast<int4*>(g + i) = lds4(s + i);
            done = n4;
        }
    }
    for (int i = done + lane; i < n; i += 32) g[i] = static_cast<Out>(s[i]);
}


// Programmatic dependent launch: the kernel is queued while its stream
// predecessor drains and waits at griddepcontrol.wait (its first statement)
// for the predecessor's results; hides the launch gap between the short
// dependent launches of small transforms.  No early trigger: a dependent
// never holds shared memory a running predecessor still needs.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// One NVTX range per launch phase (SURVEY §5 tracing): free without a tool
// attached, named phases on an nsys / ncu timeline with one.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class... KArgs, class... Args>
void launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    if (!pdl) {
        kern<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------- K1
// grid: x = row tile (S rows), y = block, z = slot (image * nq + quadrant idx)
// WsT: the pass-0 buffer's element type (wider than Acc for the int64 plans'
// pass 0 in int32, GroupLaunch::k1_acc32)
template <class In, class Acc, class Out, bool SC, class WsT = Acc>
__global__ void __launch_bounds__(kThreads, 2) k1_blocks(
    const In* __restrict__ img, int img_w, int img_h, long long img_pitch, long long img_stride, int img0, QuadSet qs,
    int W, int H,
    int ld, int S, const int4* __restrict__ blocks, const ShapeHdr* __restrict__ shapes,
    const int* __restrict__ step_offs, const PassOpDev* __restrict__ ops, const int4* __restrict__ bops, int max_width,
    int sr, int max_ops,
    WsT* __restrict__ ws, int nbuf, bool root_is_block, OutDesc out, const unsigned char* __restrict__ stage,
    long long spitch, long long simg, long long st_t, long long st_p, int pmD, int k1_ahead) {
    grid_dep_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* buf0 = reinterpret_cast<Acc*>(smem_raw);  // slots [0, max_width): parity 0
    Acc* buf1 = buf0 + (size_t)max_width * sr;     // slots [max_width, 2 max_width): parity 1

    const int tid = threadIdx.x;
    const int4 blk = blocks[blockIdx.y];
    const int x0 = blk.x;
    const ShapeHdr hdr = shapes[blk.y];
    const int wb = hdr.width, nsteps = hdr.nsteps;
    const int R = S + hdr.halo;

    const int slot = blockIdx.z;
    const int nq = qs.n;
    int img_l, qi;
    split_slot(slot, nq, img_l, qi);
    const int img_i = img0 + img_l;
    const int q = quad_code(qs, qi);
    const In* __restrict__ im = img + (size_t)img_i * img_stride;
    const int s0 = blockIdx.x * S;
    // staged pair mode: pull the leaf columns of the block `k1_ahead` CTAs
    // later in launch order into L2 (as K1P does)
    if (stage != nullptr && pmD && k1_ahead > 0 && tid == 0) {
        const long long gx = gridDim.x, gy = gridDim.y;
        const long long lin = blockIdx.x + gx * (blockIdx.y + gy * (long long)blockIdx.z) + k1_ahead;
        if (lin < gx * gy * gridDim.z) {
            const int y2 = static_cast<int>((lin / gx) % gy), z2 = static_cast<int>(lin / (gx * gy));
            int il2, qi2;
            split_slot(z2, nq, il2, qi2);
            const int q2 = quad_code(qs, qi2);
            const int4 b2 = blocks[y2];
            const int w2 = shapes[b2.y].width;
            const int cf = (q2 & 1) ? W - w2 - b2.x : b2.x;
            const unsigned char* p2 = stage + (size_t)il2 * simg + (q2 < 2 ? st_t : st_p) + (size_t)cf * spitch;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p2), "r"(static_cast<uint32_t>(w2 * spitch))
                         : "memory");
        }
    }

    // Load the tile: values of depth `nsteps` (the leaves) into buf[nsteps & 1].
    Acc* lbuf = (nsteps & 1) ? buf1 : buf0;
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int kWarps = kThreads / 32;
    if (stage != nullptr) {
        // staged u8 columns (k_stage_u8): 4 leaves per aligned 4-byte load
        const unsigned char* __restrict__ sb =
            stage + (size_t)(img_i - img0) * simg + (q < 2 ? st_t : st_p) + s0;
        const int nw = (R + 3) >> 2;
        for (int c = warp; c < wb; c += kWarps) {
            const int col = (q & 1) ? W - 1 - (x0 + c) : x0 + c;
            const uint32_t* __restrict__ cp = reinterpret_cast<const uint32_t*>(sb + (size_t)col * spitch);
            if (pmD) {  // u16 pair mode: words of rows (i, i + D)
                for (int k = lane; k < nw; k += 32)
                    sts4(lbuf + c * sr + 4 * k, pack_pair_u8x4(__ldg(cp + k), __ldg(cp + k + (pmD >> 2))));
                continue;
            }
            for (int k = lane; k < nw; k += 32) {
                const uint32_t x = __ldg(cp + k);
                sts4(lbuf + c * sr + 4 * k,
                     make_int4(to_bits<Acc>(static_cast<Acc>(x & 0xff)), to_bits<Acc>(static_cast<Acc>((x >> 8) & 0xff)),
                               to_bits<Acc>(static_cast<Acc>((x >> 16) & 0xff)), to_bits<Acc>(static_cast<Acc>(x >> 24))));
            }
        }
    } else if (q < 2) {
        // working column = image column (flipped for horiz_neg): a tile row is
        // wb contiguous image pixels.  Stage row-major (row stride wb+1, so
        // both the row writes and the column reads below are bank-conflict
        // free) in the buffer that does not receive the leaves, then
        // transpose into the column-major leaf buffer.
        Acc* stage = (nsteps & 1) ? buf0 : buf1;
        const int sw = wb + 1;
        const int xa = (q == 1) ? img_w - 1 - x0 : x0;  // image x of working column 0
        const int dx = (q == 1) ? -1 : 1;
        constexpr int kUH = 8;
        for (int ib = warp; ib < R; ib += kWarps * kUH) {
            In v[kUH][2];
#pragma unroll
            for (int u = 0; u < kUH; ++u) {
                const int i = ib + u * kWarps;
                if (i < R) {
                    const int y = s0 + R <= H ? s0 + i : wrap_any(s0 + i, H);  // tile-uniform test
                    const In* __restrict__ rowp = im + (size_t)y * img_pitch;
                    if (lane < wb) v[u][0] = rowp[xa + dx * lane];
                    if (lane + 32 < wb) v[u][1] = rowp[xa + dx * (lane + 32)];
                }
            }
#pragma unroll
            for (int u = 0; u < kUH; ++u) {
                const int i = ib + u * kWarps;
                if (i < R) {
                    if (lane < wb) stage[i * sw + lane] = static_cast<Acc>(v[u][0]);
                    if (lane + 32 < wb) stage[i * sw + lane + 32] = static_cast<Acc>(v[u][1]);
                }
            }
        }
        __syncthreads();
        for (int c = warp; c < wb; c += kWarps)
            for (int i = lane; i < R; i += 32) lbuf[c * sr + i] = stage[i * sw + c];
    } else {
        // working column = image row (reversed rows for vert_neg): contiguous.
        for (int c = warp; c < wb; c += kWarps) {
            const int row = (q == 2) ? x0 + c : img_h - 1 - (x0 + c);
            warp_load_window(lbuf + c * sr, im + (size_t)row * img_pitch, s0, R, H, lane);
        }
    }

    // Merge steps, deepest first: step k writes local depth nsteps-1-k into
    // the buffer of that parity (ops carry parity-offset slot numbers).
    for (int k = 0; k < nsteps; ++k) {
        __syncthreads();
        if constexpr (sizeof(Acc) == 4)
            run_step_baked<Acc, kWarps, SC>(smem_u32(buf0), bops + hdr.op_base, step_offs[hdr.step_base + k],
                                            step_offs[hdr.step_base + k + 1], warp, lane);
        else
            run_step<Acc, kWarps>(buf0, sr, ops + hdr.op_base, step_offs[hdr.step_base + k],
                                  step_offs[hdr.step_base + k + 1], S, warp, lane);
    }
    __syncthreads();

    // Store the block root's S rows (values of local depth 0 live in buf0).
    const int rows_out = min(S, H - s0);
    if (!root_is_block) {
        WsT* __restrict__ dstw = ws + (size_t)slot * nbuf * W * ld;  // pass 0 output: buffer 0
        const bool al = ((ld | s0) & 3) == 0;
        for (int c = warp; c < wb; c += kWarps)
            warp_store_col<Acc, WsT>(dstw + (size_t)(x0 + c) * ld + s0, buf0 + c * sr, rows_out, al, lane);
        if (pmD) {  // u16 pair mode: words [D, H) from words k and k + e of the root
            const int e = 2 * pmD - H;
            for (int c = warp; c < wb; c += kWarps) {
                const Acc* rc = buf0 + c * sr;
                WsT* __restrict__ gc = dstw + (size_t)(x0 + c) * ld + pmD;
                for (int k = lane; k < H - pmD; k += 32)
                    gc[k] = static_cast<WsT>(from_bits<Acc>(pair_extra_word(to_bits<Acc>(rc[k]), to_bits<Acc>(rc[k + e]))));
            }
        }
    } else {
        Out* o = reinterpret_cast<Out*>(out_ptr(out, q)) + (size_t)img_i * out.img_stride;
        if (out.layout == 0) {  // rows of wb contiguous slopes
            for (int i = warp; i < rows_out; i += kWarps)
                for (int c = lane; c < wb; c += 32) o[(size_t)(s0 + i) * W + c] = static_cast<Out>(buf0[c * sr + i]);
        } else {
            Out* __restrict__ pr = static_cast<Out*>(out.peer);
            for (int c = warp; c < wb; c += kWarps) {
                const bool to_peer = pr != nullptr && c >= out.peer_c0 && c < out.peer_c1;
                for (int i = lane; i < rows_out; i += 32) {
                    const Out v = static_cast<Out>(buf0[c * sr + i]);
                    o[(size_t)c * H + s0 + i] = v;
                    if (to_peer) pr[(size_t)(c - out.peer_c0) * H + s0 + i] = v;  // NVLink store
                }
            }
        }
    }
}

// --------------------------------------------------------------- staging
// u8 images -> 16-byte aligned working columns for K1P (one aligned 4-byte
// load per 4 leaves, no wrap arithmetic: rows [H, pitch) repeat rows from 0).
// One pass over 64 x 64 tiles of the (wrapped) image writes both sets:
//   T (horizontal quadrants, quadrants.cpp:34-35): T[x][y] = img[y mod h][x],
//     x < w, y < pitch_t (the tile transposed through shared memory);
//   P (vertical quadrants, quadrants.cpp:36-37): P[r][y] = img[r][y mod w],
//     r < h, y < pitch_p.
// grid: x = 64-column tiles of max(w, pitch_p), y = 64-row tiles of
// max(h, pitch_t), z = image.  16 byte loads in flight per thread.
__global__ void __launch_bounds__(256) k_stage_u8(const unsigned char* __restrict__ img, int w, int h, long long pitch,
                                                  long long img_stride, int img0, unsigned char* __restrict__ st,
                                                  long long simg, long long pitch_t, long long off_t, long long pitch_p,
                                                  long long off_p) {
    grid_dep_wait();
    __shared__ __align__(16) unsigned char tile[64][68];
    const int c0 = blockIdx.x * 64, r0 = blockIdx.y * 64, im = blockIdx.z;
    const bool want_t = off_t >= 0 && c0 < w && r0 < pitch_t;
    const bool want_p = off_p >= 0 && r0 < h && c0 < pitch_p;
    if (!want_t && !want_p) return;
    const unsigned char* __restrict__ base = img + (size_t)(img0 + im) * img_stride;
    // a tile wholly past column w holds wrapped columns c0 - w.. (the P set)
    const int cs0 = c0 < w ? c0 : c0 - w;
    if (cs0 + 64 <= w && (c0 < w || c0 - w < w)) {
        // columns in range (rows may wrap: the staged columns run past h):
        // each row segment read as aligned 4-byte words (two per 4 pixels,
        // funnel-shifted into place), 4 words per thread
        const int j = threadIdx.x & 15, rr0 = threadIdx.x >> 4;  // word j of rows rr0, rr0 + 16, ...
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int r = r0 + rr0 + 16 * k;
            if (r >= h) r = r - h < h ? r - h : r % h;  // the wrapped head rows
            const unsigned char* p = base + (size_t)r * pitch + cs0 + 4 * j;
            const uint32_t* a = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
            const uint32_t sh = 8u * static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p) & 3);
            v[k] = __funnelshift_r(__ldg(a), sh ? __ldg(a + 1) : 0u, sh);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) *reinterpret_cast<uint32_t*>(&tile[rr0 + 16 * k][4 * j]) = v[k];
    } else {
        const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
        int c = c0 + tx;
        if (c >= w) c = c - w < w ? c - w : c % w;
        const unsigned char* __restrict__ src = base + c;
        unsigned char v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int r = r0 + ty + 4 * k;
            if (r >= h) r = r - h < h ? r - h : r % h;  // the wrapped head rows
            v[k] = src[(size_t)r * pitch];
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) tile[ty + 4 * k][tx] = v[k];
    }
    __syncthreads();
    unsigned char* __restrict__ dst = st + (size_t)im * simg;
    if (want_t) {
        // thread = a 4 x 4 byte block (rows 4j.., columns 4i..): four aligned
        // word reads, a byte transpose, four T words (lanes along j: each
        // group of 16 lanes writes 64 contiguous bytes of one T column)
        const int j = threadIdx.x & 15, i = threadIdx.x >> 4;
        const uint32_t a = *reinterpret_cast<const uint32_t*>(&tile[4 * j][4 * i]);
        const uint32_t b = *reinterpret_cast<const uint32_t*>(&tile[4 * j + 1][4 * i]);
        const uint32_t cc = *reinterpret_cast<const uint32_t*>(&tile[4 * j + 2][4 * i]);
        const uint32_t d = *reinterpret_cast<const uint32_t*>(&tile[4 * j + 3][4 * i]);
        const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
        const uint32_t t2 = __byte_perm(cc, d, 0x5140), t3 = __byte_perm(cc, d, 0x7362);
        const uint32_t col[4] = {__byte_perm(t0, t2, 0x5410), __byte_perm(t0, t2, 0x7632), __byte_perm(t1, t3, 0x5410),
                                 __byte_perm(t1, t3, 0x7632)};
        const long long y = r0 + 4 * j;
        if (y < pitch_t) {
            unsigned char* __restrict__ tp = dst + off_t + (size_t)(c0 + 4 * i) * pitch_t + y;
#pragma unroll
            for (int m = 0; m < 4; ++m, tp += pitch_t)
                if (c0 + 4 * i + m < w) *reinterpret_cast<uint32_t*>(tp) = col[m];
        }
    }
    if (want_p) {  // word j of P row r = r0 + rr: columns c0 + 4j .. + 3
        const int j = threadIdx.x & 15, rr0 = threadIdx.x >> 4;
        const long long y = c0 + 4 * j;
        if (y < pitch_p) {
            unsigned char* __restrict__ pp = dst + off_p + (size_t)(r0 + rr0) * pitch_p + y;
            const size_t pstep = 16 * (size_t)pitch_p;
#pragma unroll
            for (int k = 0; k < 4; ++k, pp += pstep)
                if (r0 + rr0 + 16 * k < h)
                    *reinterpret_cast<uint32_t*>(pp) = *reinterpret_cast<const uint32_t*>(&tile[rr0 + 16 * k][4 * j]);
        }
    }
}

// ------------------------------------------------------------------ K1P
// Specialised pass 0 for the common block: a width-32 Brady-Yong subtree
// (every power-of-two block; all but at most one block of a Tweaked tree).
// Its ops need no tables: (t0, t1, shift) follow from the column index with
// a compile-time divisor per level.  512 threads; warp w owns columns w and w + 16 at every
// level.  Levels 1-2 run in registers (lanes own 4-row vectors, whose shifted
// neighbours the level-2 outputs share); levels 3-5 interleave rows over
// lanes so every shift is conflict-free.  Leaves live in slots [32, 64); the
// levels alternate parity and the block root ends in slots [32, 64).
constexpr int kBYW = 32;        // block width
constexpr int kBYMaxS = 256;    // rows per tile (host guarantees S <= 256)
constexpr int kBYSR = 300;      // slot stride: >= 256 + 31 + 12, multiple of 4, /4 odd
constexpr int kThreadsBY = 512;
static_assert(kThreadsBY == 8 * 64, "levels 1-2 map 8 column groups x 64 threads");
constexpr int kWarpsBY = kThreadsBY / 32;
// K1P on 576 threads: 8 column groups x 72 threads take the 71 level-2 row
// chunks of a 256-row tile in one round (with 512 threads, 7 of each group's
// 64 threads ran a second item that the whole CTA then waited for); the
// leaves and levels 3-5 stay on warps 0-15.  56 registers keep two CTAs/SM.
constexpr int kThreadsBYP = 576;

// Level L (1..5) merges widths 2^(L-1) -> 2^L.  For block-local column T
// the children's slope t0 = t1 = rhu(tl (w0-1), w-1) (split.hpp:53-57) is
// computed arithmetically (the divisor is a compile-time constant), so all
// warps run the same short code path (no per-warp unrolled tables: those
// thrashed the instruction cache).  Only the 4 residues of the shift are
// specialised.
// Variant 0 of a K1P op: C++ shared pointers, 3 predicated 128-row chunks.
template <int M, class Acc>
__device__ __forceinline__ void by_rows(Acc* __restrict__ d, const Acc* __restrict__ a, const Acc* __restrict__ bb,
                                        int n, int lane) {
    int4 av[3], b0[3], b1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        if (lane * 4 + 128 * c < n) {
            av[c] = lds4(a + 128 * c);
            b0[c] = lds4(bb + 128 * c);
            if (M) b1[c] = lds4(bb + 128 * c + 4);
        }
#pragma unroll
    for (int c = 0; c < 3; ++c)
        if (lane * 4 + 128 * c < n) sts4(d + 128 * c, add_shift<M, Acc>(av[c], b0[c], M ? b1[c] : b0[c]));
}

// Levels 3-5, rows interleaved over lanes (lane l owns rows l, l+32, ...):
// any shift is one conflict-free wavefront per 32 rows (n <= 256 + 31).
template <class Acc, int L, int F = 0, int SF = 0>
__device__ __forceinline__ void by_level_s(Acc* sm, int S, int warp, int lane) {
    constexpr int w = 1 << L, w0 = w >> 1;
    constexpr int src = ((7 - L + F) & 1) * kBYW, dst = ((6 - L + F) & 1) * kBYW;
    constexpr int G = (kBYMaxS + kBYW + 31) / 32;  // 9 row groups at most
    // SF: the row tile known at compile time (the full 256-row tiles): the
    // row-group predicates of all but the last group fold away
    const int n = (SF ? SF : S) + kBYW - w;
    const uint32_t base = smem_u32(sm) + lane * 4u;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        const int T = warp + h * kWarpsBY;
        const int tl = T & (w - 1), x0 = T & ~(w - 1);
        const int t0 = (2 * tl * (w0 - 1) + (w - 1)) / (2 * (w - 1));
        const int r = tl - t0;
        const uint32_t d = base + (dst + T) * kBYSR * 4u;
        const uint32_t a = base + (src + x0 + t0) * kBYSR * 4u;
        const uint32_t b = base + ((src + x0 + w0 + t0) * kBYSR + r) * 4u;
        int x[G], y[G];
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (32 * u + lane < n) {
                x[u] = lds1u(a + 128u * u);
                y[u] = lds1u(b + 128u * u);
            }
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (32 * u + lane < n) sts1u(d + 128u * u, add_bits<Acc>(x[u], y[u]));
    }
}

// Levels 3, 4 (shared memory, rows interleaved over lanes) and 5 (stored
// from registers); full 256-row tiles take the compile-time row count.
template <class Acc, class WsT = Acc>
__device__ __forceinline__ void by_levels_345(Acc* sm, int S, int warp, int lane, WsT* __restrict__ dcol0, int ld,
                                              int rows_out, bool act = true);

// Level 5 (the block root) written straight to the pass-0 buffer from
// registers: lane = row, so each warp store is 32 consecutive rows of one
// column (coalesced), and the root never round-trips through shared memory.
// WsT: the pass-0 buffer's element type (int64 for the int64 plans' pass 0
// in int32, see GroupLaunch::k1_acc32): the block root widened on the store.
template <class Acc, int SF = 0, class WsT = Acc>
__device__ __forceinline__ void by_level5_store(Acc* sm, int S, int warp, int lane, WsT* __restrict__ dcol0, int ld,
                                                int rows_out_) {
    const int rows_out = SF ? SF : rows_out_;  // SF: a full tile, rows known at compile time
    constexpr int w = 32, w0 = 16;
    constexpr int src = 0;  // level 4 output (parity of V3): slots [0, 32)
    constexpr int G = (kBYMaxS + 31) / 32;
    const uint32_t base = smem_u32(sm) + lane * 4u;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        const int T = warp + h * kWarpsBY;
        const int t0 = (2 * T * (w0 - 1) + (w - 1)) / (2 * (w - 1));
        const int r = T - t0;
        const uint32_t a = base + (src + t0) * kBYSR * 4u;
        const uint32_t b = base + ((src + w0 + t0) * kBYSR + r) * 4u;
        WsT* __restrict__ g = dcol0 + (size_t)T * ld + lane;
        int x[G], y[G];
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (32 * u + lane < rows_out) {
                x[u] = lds1u(a + 128u * u);
                y[u] = lds1u(b + 128u * u);
            }
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (32 * u + lane < rows_out) g[32 * u] = static_cast<WsT>(from_bits<Acc>(add_bits<Acc>(x[u], y[u])));
    }
}

template <class Acc, class WsT>
__device__ __forceinline__ void by_levels_345(Acc* sm, int S, int warp, int lane, WsT* __restrict__ dcol0, int ld,
                                              int rows_out, bool act) {
    if (S == kBYMaxS) {
        if (act) by_level_s<Acc, 3, 0, kBYMaxS>(sm, S, warp, lane);
        __syncthreads();
        if (act) by_level_s<Acc, 4, 0, kBYMaxS>(sm, S, warp, lane);  // -> slots [0, 32)
    } else {
        if (act) by_level_s<Acc, 3>(sm, S, warp, lane);
        __syncthreads();
        if (act) by_level_s<Acc, 4>(sm, S, warp, lane);
    }
    __syncthreads();
    if (!act) return;
    if (rows_out == kBYMaxS)  // a full tile (the last row tile may be shorter)
        by_level5_store<Acc, kBYMaxS, WsT>(sm, S, warp, lane, dcol0, ld, rows_out);
    else
        by_level5_store<Acc, 0, WsT>(sm, S, warp, lane, dcol0, ld, rows_out);
}

template <class Acc, int L, int F = 0>
__device__ __forceinline__ void by_level_v0(Acc* sm, int S, int warp, int lane) {
    constexpr int w = 1 << L, w0 = w >> 1;
    constexpr int src = ((6 - L + F) & 1) * kBYW, dst = ((5 - L + F) & 1) * kBYW;
    const int n = S + kBYW - w;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int T = warp + h * kWarpsBY;
        const int tl = T & (w - 1), x0 = T & ~(w - 1);
        const int t0 = (2 * tl * (w0 - 1) + (w - 1)) / (2 * (w - 1));
        const int r = tl - t0;
        Acc* d = sm + (dst + T) * kBYSR + lane * 4;
        const Acc* a = sm + (src + x0 + t0) * kBYSR + lane * 4;
        const Acc* bb = sm + (src + x0 + w0 + t0) * kBYSR + (r & ~3) + lane * 4;
        switch (r & 3) {
            case 0: by_rows<0>(d, a, bb, n, lane); break;
            case 1: by_rows<1>(d, a, bb, n, lane); break;
            case 2: by_rows<2>(d, a, bb, n, lane); break;
            default: by_rows<3>(d, a, bb, n, lane); break;
        }
    }
}

// Levels 1 and 2 of a width-32 block fused in registers: item (g, j) reads
// the leaves of columns 4g..4g+3, rows 4j..4j+7 (two aligned 16-byte loads
// per column), forms both level-1 pairs (shift 0/1) and the level-2 width-4
// merge (t0 = 0,0,1,1; shift 0,1,1,2 -- BYOp at L = 1, 2) and stores rows
// 4j..4j+3 of the 4 level-2 columns.  Leaves: slots [32, 64); level 2: slots
// [0, 32).  Rows produced: [0, S + 28) (the halo levels 3..5 still need).
template <class Acc>
__device__ __forceinline__ int4 add4(int4 a, int4 b) {
    return make_int4(to_bits<Acc>(from_bits<Acc>(a.x) + from_bits<Acc>(b.x)),
                     to_bits<Acc>(from_bits<Acc>(a.y) + from_bits<Acc>(b.y)),
                     to_bits<Acc>(from_bits<Acc>(a.z) + from_bits<Acc>(b.z)),
                     to_bits<Acc>(from_bits<Acc>(a.w) + from_bits<Acc>(b.w)));
}
// rows k..k+3 of a column held as two vectors (rows 0..3, 4..7) shifted by K
template <int K>
__device__ __forceinline__ int4 shifted(int4 lo, int4 hi) {
    const int v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    return make_int4(v[K], v[K + 1], v[K + 2], v[K + 3]);
}

template <class Acc, int GT = 64>
__device__ __forceinline__ void by_level12(Acc* sm, int S, int tid) {
    const int nchunk = (S + kBYW - 4 + 3) >> 2;  // row chunks of 4 the level-2 output needs
    const int4* V = reinterpret_cast<const int4*>(sm);
    int4* O = reinterpret_cast<int4*>(sm);
    constexpr int s4 = kBYSR / 4;
    const int g = tid / GT;  // 8 column groups x GT threads; lanes over row chunks: conflict-free
    for (int j = tid - g * GT; j < nchunk; j += GT) {
        const int c0 = (kBYW + 4 * g) * s4 + j;  // leaves of column 4g, chunk j
        // pair (4g, 4g+1) -> level-1 columns p0 (shift 0), p1 (shift 1), rows j*4 .. j*4+6
        const int4 a0 = V[c0], a1 = V[c0 + 1], b0 = V[c0 + s4], b1 = V[c0 + s4 + 1];
        const int4 e0 = V[c0 + 2 * s4], e1 = V[c0 + 2 * s4 + 1], f0 = V[c0 + 3 * s4], f1 = V[c0 + 3 * s4 + 1];
        // level 1 (rows 0..3 and 4..7 of each output, from the two vectors)
        const int4 p0l = add4<Acc>(a0, b0), p0h = add4<Acc>(a1, b1);
        const int4 p1l = add4<Acc>(a0, shifted<1>(b0, b1)), p1h = add4<Acc>(a1, shifted<1>(b1, b1));
        const int4 q0l = add4<Acc>(e0, f0), q0h = add4<Acc>(e1, f1);
        const int4 q1l = add4<Acc>(e0, shifted<1>(f0, f1)), q1h = add4<Acc>(e1, shifted<1>(f1, f1));
        // level 2: o0 = p0 + q0, o1 = p0 + q0[+1], o2 = p1 + q1[+1], o3 = p1 + q1[+2]
        const int d0 = (4 * g) * s4 + j;
        O[d0] = add4<Acc>(p0l, q0l);
        O[d0 + s4] = add4<Acc>(p0l, shifted<1>(q0l, q0h));
        O[d0 + 2 * s4] = add4<Acc>(p1l, shifted<1>(q1l, q1h));
        O[d0 + 3 * s4] = add4<Acc>(p1l, shifted<2>(q1l, q1h));
        (void)p0h;
        (void)p1h;
    }
}

// Levels 1-2 straight from the staged u8 columns (k_stage_u8): the same
// items as by_level12, the leaf vectors unpacked from aligned 4-byte global
// loads (lanes over consecutive row chunks: coalesced) instead of a leaf
// tile in shared memory -- the leaves never touch shared memory.
template <class Acc>
__device__ __forceinline__ int4 unpack_u8x4(uint32_t x) {
    return make_int4(to_bits<Acc>(static_cast<Acc>(x & 0xff)), to_bits<Acc>(static_cast<Acc>((x >> 8) & 0xff)),
                     to_bits<Acc>(static_cast<Acc>((x >> 16) & 0xff)), to_bits<Acc>(static_cast<Acc>(x >> 24)));
}
template <class Acc, int GT = 64>
__device__ __forceinline__ void by_level12_staged(Acc* sm, int S, int tid, const unsigned char* __restrict__ sb,
                                                  long long spitch, int W, int x0, bool rev) {
    const int nchunk = (S + kBYW - 4 + 3) >> 2;
    int4* O = reinterpret_cast<int4*>(sm);
    constexpr int s4 = kBYSR / 4;
    const int g = tid / GT;  // 8 column groups x GT threads, lanes over consecutive row chunks
    for (int j = tid - g * GT; j < nchunk; j += GT) {
        const int c = x0 + 4 * g;
        const long long cs = rev ? -spitch : spitch;  // reversed column order for horiz_neg / vert_neg
        const unsigned char* pa = sb + (long long)(rev ? W - 1 - c : c) * spitch + 4 * j;
        const uint32_t* A = reinterpret_cast<const uint32_t*>(pa);
        const uint32_t* B = reinterpret_cast<const uint32_t*>(pa + cs);
        const uint32_t* E = reinterpret_cast<const uint32_t*>(pa + 2 * cs);
        const uint32_t* F = reinterpret_cast<const uint32_t*>(pa + 3 * cs);
        const uint32_t wa0 = __ldg(A), wb0 = __ldg(B), wb1 = __ldg(B + 1), we0 = __ldg(E), we1 = __ldg(E + 1),
                       wf0 = __ldg(F), wf1 = __ldg(F + 1);
        const int4 a0 = unpack_u8x4<Acc>(wa0), b0 = unpack_u8x4<Acc>(wb0), b1 = unpack_u8x4<Acc>(wb1);
        const int4 e0 = unpack_u8x4<Acc>(we0), e1 = unpack_u8x4<Acc>(we1), f0 = unpack_u8x4<Acc>(wf0),
                   f1 = unpack_u8x4<Acc>(wf1);
        const int4 p0l = add4<Acc>(a0, b0);
        const int4 p1l = add4<Acc>(a0, shifted<1>(b0, b1));
        const int4 q0l = add4<Acc>(e0, f0), q0h = add4<Acc>(e1, f1);
        const int4 q1l = add4<Acc>(e0, shifted<1>(f0, f1)), q1h = add4<Acc>(e1, shifted<1>(f1, f1));
        const int d0 = (4 * g) * s4 + j;
        O[d0] = add4<Acc>(p0l, q0l);
        O[d0 + s4] = add4<Acc>(p0l, shifted<1>(q0l, q0h));
        O[d0 + 2 * s4] = add4<Acc>(p1l, shifted<1>(q1l, q1h));
        O[d0 + 3 * s4] = add4<Acc>(p1l, shifted<2>(q1l, q1h));
    }
}

// by_level12_staged in the u16 pair mode: the leaf words pack rows 4j.. of
// the low half with rows 4j + D.. of the high half (both aligned: D % 4 == 0).
template <class Acc, int GT = 64>
__device__ __forceinline__ void by_level12_staged_pair(Acc* sm, int S, int tid, const unsigned char* __restrict__ sb,
                                                       long long spitch, int W, int x0, bool rev, int D) {
    const int nchunk = (S + kBYW - 4 + 3) >> 2;
    int4* O = reinterpret_cast<int4*>(sm);
    constexpr int s4 = kBYSR / 4;
    const int g = tid / GT;  // GT threads per 4-column group
    const int dw = D >> 2;  // the high half, in 4-byte words
    for (int j = tid - g * GT; j < nchunk; j += GT) {
        const int c = x0 + 4 * g;
        const long long cs = rev ? -spitch : spitch;
        const unsigned char* pa = sb + (long long)(rev ? W - 1 - c : c) * spitch + 4 * j;
        const uint32_t* A = reinterpret_cast<const uint32_t*>(pa);
        const uint32_t* B = reinterpret_cast<const uint32_t*>(pa + cs);
        const uint32_t* E = reinterpret_cast<const uint32_t*>(pa + 2 * cs);
        const uint32_t* F = reinterpret_cast<const uint32_t*>(pa + 3 * cs);
        const uint32_t wa0 = __ldg(A), wb0 = __ldg(B), wb1 = __ldg(B + 1), we0 = __ldg(E), we1 = __ldg(E + 1),
                       wf0 = __ldg(F), wf1 = __ldg(F + 1);
        const uint32_t ha0 = __ldg(A + dw), hb0 = __ldg(B + dw), hb1 = __ldg(B + dw + 1), he0 = __ldg(E + dw),
                       he1 = __ldg(E + dw + 1), hf0 = __ldg(F + dw), hf1 = __ldg(F + dw + 1);
        const int4 a0 = pack_pair_u8x4(wa0, ha0), b0 = pack_pair_u8x4(wb0, hb0), b1 = pack_pair_u8x4(wb1, hb1);
        const int4 e0 = pack_pair_u8x4(we0, he0), e1 = pack_pair_u8x4(we1, he1), f0 = pack_pair_u8x4(wf0, hf0),
                   f1 = pack_pair_u8x4(wf1, hf1);
        const int4 p0l = add4<Acc>(a0, b0);
        const int4 p1l = add4<Acc>(a0, shifted<1>(b0, b1));
        const int4 q0l = add4<Acc>(e0, f0), q0h = add4<Acc>(e1, f1);
        const int4 q1l = add4<Acc>(e0, shifted<1>(f0, f1)), q1h = add4<Acc>(e1, shifted<1>(f1, f1));
        const int d0 = (4 * g) * s4 + j;
        O[d0] = add4<Acc>(p0l, q0l);
        O[d0 + s4] = add4<Acc>(p0l, shifted<1>(q0l, q0h));
        O[d0 + 2 * s4] = add4<Acc>(p1l, shifted<1>(q1l, q1h));
        O[d0 + 3 * s4] = add4<Acc>(p1l, shifted<2>(q1l, q1h));
    }
}

// Level 5 of the pair mode: words [0, D) stored from registers as in
// by_level5_store, then words [D, H) formed with one lane shuffle per group:
// the source lane pre-selects the group the requesting lane needs (a lane
// below e serves the next group's wrap-around).  DC: D known at compile time.
template <class Acc, int DC = 0>
__device__ __forceinline__ void by_level5_store_pair(Acc* sm, int warp, int lane, Acc* __restrict__ dcol0, int ld,
                                                     int D_, int H) {
    constexpr int w = 32, w0 = 16;
    constexpr int G = kBYMaxS / 32;  // D <= 256
    const int D = DC ? DC : D_;
    const int e = 2 * D - H, nx = H - D;
    const int sl = (lane + e) & 31;
    const bool wrap_src = lane < e;  // this lane's word is wanted by lane + 32 - e of the previous group
    const uint32_t base = smem_u32(sm) + lane * 4u;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        const int T = warp + h * kWarpsBY;
        const int t0 = (2 * T * (w0 - 1) + (w - 1)) / (2 * (w - 1));
        const int r = T - t0;
        const uint32_t a = base + t0 * kBYSR * 4u;
        const uint32_t b = base + ((w0 + t0) * kBYSR + r) * 4u;
        Acc* __restrict__ g = dcol0 + (size_t)T * ld + lane;
        int x[G], y[G], v[G + 1];
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (32 * u + lane < D) {
                x[u] = lds1u(a + 128u * u);
                y[u] = lds1u(b + 128u * u);
            }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            v[u] = 32 * u + lane < D ? add_bits<Acc>(x[u], y[u]) : 0;
            if (32 * u + lane < D) g[32 * u] = from_bits<Acc>(v[u]);
        }
        v[G] = 0;
#pragma unroll
        for (int u = 0; u < G; ++u) {
            if (32 * u >= nx) break;  // warp-uniform
            const int hi = __shfl_sync(0xffffffffu, wrap_src ? v[u + 1] : v[u], sl);
            if (32 * u + lane < nx) g[D + 32 * u] = from_bits<Acc>(pair_extra_word(v[u], hi));
        }
    }
}

// grid: x = row tile, y = BY-32 block, z = slot.  Writes pass-0 buffer 0.
template <class In, class Acc, int V, int NT = kThreadsBY, class WsT = Acc>
__global__ void __launch_bounds__(NT, 2) k1_by32(const In* __restrict__ img, int img_w, int img_h,
                                                          long long img_pitch, long long img_stride, int img0, QuadSet qs, int W, int H,
                                                          int ld, int S, const int* __restrict__ bx0,
                                                          WsT* __restrict__ ws, int nbuf,
                                                          const unsigned char* __restrict__ stage, long long spitch,
                                                          long long simg, long long st_t, long long st_p, int pmD) {
    grid_dep_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* sm = reinterpret_cast<Acc*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int x0 = bx0[blockIdx.y];
    const int slot = blockIdx.z;
    const int nq = qs.n;
    int img_l, qi;
    split_slot(slot, nq, img_l, qi);
    const int img_i = img0 + img_l;
    const int q = quad_code(qs, qi);
    const In* __restrict__ im = img + (size_t)img_i * img_stride;
    const int s0 = blockIdx.x * S;
    const int R = S + kBYW - 1;
    Acc* leaves = sm + kBYW * kBYSR;  // parity 1
    constexpr int kRowsPerLane = (kBYMaxS + kBYW - 1 + 31) / 32;  // 9
    static_assert(NT == kThreadsBY || (NT == kThreadsBYP && V == 5), "576 threads: variant 5 only");
    static_assert(std::is_same<WsT, Acc>::value || V == 5, "a widening pass-0 store: variant 5 only");
    const bool act = NT == kThreadsBY || warp < kWarpsBY;  // the warps that own columns
    if (V == 5 && stage != nullptr) {
        // levels 1-2 read the staged columns directly (no leaf tile)
        const unsigned char* __restrict__ sb =
            stage + (size_t)(img_i - img0) * simg + (q < 2 ? st_t : st_p) + s0;
        if (NT == kThreadsBY && pmD) {  // u16 pair mode: one tile of words [0, D), S == D
            by_level12_staged_pair<Acc>(sm, S, tid, sb, spitch, W, x0, (q & 1) != 0, pmD);
            __syncthreads();
            if (S == kBYMaxS) {
                by_level_s<Acc, 3, 0, kBYMaxS>(sm, S, warp, lane);
                __syncthreads();
                by_level_s<Acc, 4, 0, kBYMaxS>(sm, S, warp, lane);
            } else {
                by_level_s<Acc, 3>(sm, S, warp, lane);
                __syncthreads();
                by_level_s<Acc, 4>(sm, S, warp, lane);
            }
            __syncthreads();
            if constexpr (std::is_same<WsT, Acc>::value) {
                Acc* __restrict__ dcol0 = ws + (size_t)slot * nbuf * W * ld + (size_t)x0 * ld;
                if (pmD == kBYMaxS) by_level5_store_pair<Acc, kBYMaxS>(sm, warp, lane, dcol0, ld, pmD, H);
                else by_level5_store_pair<Acc>(sm, warp, lane, dcol0, ld, pmD, H);
            }
            return;
        }
        by_level12_staged<Acc, NT / 8>(sm, S, tid, sb, spitch, W, x0, (q & 1) != 0);
        __syncthreads();
        by_levels_345<Acc, WsT>(sm, S, warp, lane, ws + (size_t)slot * nbuf * W * ld + (size_t)x0 * ld + s0, ld,
                           min(S, H - s0), act);
        return;
    }
    if (!act) {
        // warps 16.. of a 576-thread CTA: no leaves to load (the q < 2 path
        // has one barrier)
        if (q < 2 && stage == nullptr) __syncthreads();
    } else if (stage != nullptr) {
        // staged u8 columns (k_stage_t/p): 4 leaves per aligned 4-byte load,
        // one 16-byte shared store (lanes contiguous: conflict-free)
        const unsigned char* __restrict__ sb =
            stage + (size_t)(img_i - img0) * simg + (q < 2 ? st_t : st_p) + s0;
        const int nw = (R + 3) >> 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = warp + h * kWarpsBY;
            const int col = (q & 1) ? W - 1 - (x0 + c) : x0 + c;
            const uint32_t* __restrict__ cp = reinterpret_cast<const uint32_t*>(sb + (size_t)col * spitch);
            uint32_t v[3];
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (lane + 32 * k < nw) v[k] = __ldg(cp + lane + 32 * k);
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (lane + 32 * k < nw) {
                    const uint32_t x = v[k];
                    sts4(leaves + c * kBYSR + 4 * (lane + 32 * k),
                         make_int4(to_bits<Acc>(static_cast<Acc>(x & 0xff)), to_bits<Acc>(static_cast<Acc>((x >> 8) & 0xff)),
                                   to_bits<Acc>(static_cast<Acc>((x >> 16) & 0xff)),
                                   to_bits<Acc>(static_cast<Acc>(x >> 24))));
                }
        }
    } else if (q < 2) {
        // image rows: 32 contiguous pixels per tile row; stage row-major
        // (stride 33, conflict-free both ways) in parity 0, then transpose.
        Acc* stage = sm;
        const int xx = (q == 1) ? img_w - 1 - (x0 + lane) : x0 + lane;
        constexpr int kRowsPerWarp = (kBYMaxS + kBYW - 1 + kWarpsBY - 1) / kWarpsBY;  // 18
        In v[kRowsPerWarp];
        if (s0 + R <= H) {  // no wrap in this row tile (all but the last): one pointer stride
            const In* __restrict__ p = im + (size_t)(s0 + warp) * img_pitch + xx;
            const size_t step = (size_t)kWarpsBY * img_pitch;
#pragma unroll
            for (int k = 0; k < kRowsPerWarp; ++k)
                if (warp + k * kWarpsBY < R) v[k] = p[k * step];
        } else {
#pragma unroll
            for (int k = 0; k < kRowsPerWarp; ++k) {
                const int i = warp + k * kWarpsBY;
                if (i < R) v[k] = im[(size_t)wrap_any(s0 + i, H) * img_pitch + xx];
            }
        }
#pragma unroll
        for (int k = 0; k < kRowsPerWarp; ++k) {
            const int i = warp + k * kWarpsBY;
            if (i < R) stage[i * 33 + lane] = static_cast<Acc>(v[k]);
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = warp + h * kWarpsBY;
#pragma unroll
            for (int k = 0; k < kRowsPerLane; ++k) {
                const int i = lane + 32 * k;
                if (i < R) leaves[c * kBYSR + i] = stage[i * 33 + c];
            }
        }
    } else {
        // image rows are working columns: contiguous windows, 18 loads in flight per lane
        In v[2][kRowsPerLane];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = warp + h * kWarpsBY;
            const int row = (q == 2) ? x0 + c : img_h - 1 - (x0 + c);
            const In* __restrict__ rp = im + (size_t)row * img_pitch;
            if (s0 + R <= H) {  // no wrap in this row tile
#pragma unroll
                for (int k = 0; k < kRowsPerLane; ++k)
                    if (lane + 32 * k < R) v[h][k] = rp[s0 + lane + 32 * k];
            } else {
#pragma unroll
                for (int k = 0; k < kRowsPerLane; ++k) {
                    const int i = lane + 32 * k;
                    if (i < R) v[h][k] = rp[wrap_any(s0 + i, H)];
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = warp + h * kWarpsBY;
#pragma unroll
            for (int k = 0; k < kRowsPerLane; ++k) {
                const int i = lane + 32 * k;
                if (i < R) leaves[c * kBYSR + i] = static_cast<Acc>(v[h][k]);
            }
        }
    }
    __syncthreads();
    if constexpr (V >= 4) {  // (V = 5 without staging lands here)
        by_level12<Acc, NT / 8>(sm, S, tid);  // levels 1-2 in registers -> slots [0, 32)
        __syncthreads();
        by_levels_345<Acc, WsT>(sm, S, warp, lane, ws + (size_t)slot * nbuf * W * ld + (size_t)x0 * ld + s0, ld,
                           min(S, H - s0), act);
        return;
    } else if constexpr (V == 3) {
        by_level12<Acc>(sm, S, tid);  // levels 1-2 in registers -> slots [0, 32)
        __syncthreads();
        by_level_s<Acc, 3>(sm, S, warp, lane);
        __syncthreads();
        by_level_s<Acc, 4>(sm, S, warp, lane);
        __syncthreads();
        by_level_s<Acc, 5>(sm, S, warp, lane);  // block root -> slots [32, 64)
    } else if constexpr (V == 2) {
        by_level12<Acc>(sm, S, tid);  // levels 1-2 in registers -> slots [0, 32)
        __syncthreads();
        by_level_v0<Acc, 3, 1>(sm, S, warp, lane);
        __syncthreads();
        by_level_v0<Acc, 4, 1>(sm, S, warp, lane);
        __syncthreads();
        by_level_v0<Acc, 5, 1>(sm, S, warp, lane);  // block root -> slots [32, 64)
    } else {
        by_level_v0<Acc, 1>(sm, S, warp, lane);
        __syncthreads();
        by_level_v0<Acc, 2>(sm, S, warp, lane);
        __syncthreads();
        by_level_v0<Acc, 3>(sm, S, warp, lane);
        __syncthreads();
        by_level_v0<Acc, 4>(sm, S, warp, lane);
        __syncthreads();
        by_level_v0<Acc, 5>(sm, S, warp, lane);
    }
    __syncthreads();
    const int rows_out = min(S, H - s0);
    WsT* __restrict__ dstw = ws + (size_t)slot * nbuf * W * ld;
    const bool al = ((ld | s0) & 3) == 0;
    const Acc* root = sm + (V >= 2 ? kBYW * kBYSR : 0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = warp + h * kWarpsBY;
        warp_store_col<Acc, WsT>(dstw + (size_t)(x0 + c) * ld + s0, root + c * kBYSR, rows_out, al, lane);
    }
}

// K1P of the u16 pair mode on 576 threads (kThreadsBYP): levels 3-5 run on
// warps 0-15 as in k1_by32.
template <class Acc>
__global__ void __launch_bounds__(kThreadsBYP, 2) k1_by32_pair(QuadSet qs, int W, int H, int ld, int S,
                                                                const int* __restrict__ bx0, Acc* __restrict__ ws,
                                                                int nbuf, const unsigned char* __restrict__ stage,
                                                                long long spitch, long long simg, long long st_t,
                                                                long long st_p, int pmD, int ahead) {
    grid_dep_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* sm = reinterpret_cast<Acc*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int x0 = bx0[blockIdx.y];
    const int slot = blockIdx.z;
    int img_l, qi;
    split_slot(slot, qs.n, img_l, qi);
    const int q = quad_code(qs, qi);
    const unsigned char* __restrict__ sb = stage + (size_t)img_l * simg + (q < 2 ? st_t : st_p);
    // The staged leaf columns of the block `ahead` CTAs later in launch order
    // (about one wave: the CTA that will take this SM slot next) are pulled
    // into L2 by one TMA prefetch, so that CTA's leaf loads hit L2 instead of
    // waiting on DRAM (the loads are K1P's largest stall).
    if (ahead > 0 && tid == 0) {
        const long long lin = blockIdx.y + (long long)gridDim.y * blockIdx.z + ahead;
        if (lin < (long long)gridDim.y * gridDim.z) {
            const int y2 = static_cast<int>(lin % gridDim.y), z2 = static_cast<int>(lin / gridDim.y);
            int img2, qi2;
            split_slot(z2, qs.n, img2, qi2);
            const int q2 = quad_code(qs, qi2);
            const int c0 = bx0[y2];
            const int cf = (q2 & 1) ? W - kBYW - c0 : c0;  // the first column in memory (reversed sets)
            const unsigned char* p2 = stage + (size_t)img2 * simg + (q2 < 2 ? st_t : st_p) + (size_t)cf * spitch;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p2),
                         "r"(static_cast<uint32_t>(kBYW * spitch)) : "memory");
        }
    }
    by_level12_staged_pair<Acc, kThreadsBYP / 8>(sm, S, tid, sb, spitch, W, x0, (q & 1) != 0, pmD);
    __syncthreads();
    if (warp < kWarpsBY) {
        if (S == kBYMaxS) by_level_s<Acc, 3, 0, kBYMaxS>(sm, S, warp, lane);
        else by_level_s<Acc, 3>(sm, S, warp, lane);
    }
    __syncthreads();
    if (warp < kWarpsBY) {
        if (S == kBYMaxS) by_level_s<Acc, 4, 0, kBYMaxS>(sm, S, warp, lane);
        else by_level_s<Acc, 4>(sm, S, warp, lane);
    }
    __syncthreads();
    if (warp < kWarpsBY) {
        Acc* __restrict__ dcol0 = ws + (size_t)slot * nbuf * W * ld + (size_t)x0 * ld;
        if (pmD == kBYMaxS) by_level5_store_pair<Acc, kBYMaxS>(sm, warp, lane, dcol0, ld, pmD, H);
        else by_level5_store_pair<Acc>(sm, warp, lane, dcol0, ld, pmD, H);
    }
}

size_t k1_by32_smem_bytes() { return (2 * kBYW * kBYSR + 16) * 4; }

// ------------------------------------------------------------------- K2
// One fused upper pass.  grid: x = row tile (S rows), y = tile (G slopes of
// one band node), z = slot (image * nq + quadrant index).  A tile is a small
// program (plan.cpp build_tile): load the row windows of the frontier columns
// it depends on, run its merge ops level by level in shared memory (slot-
// major, row capacity L), then store its G columns -- into the other
// workspace buffer, or (root pass) straight into the output in the
// reference layout hough[s*W + t] (transform.cpp:80-83).
constexpr int kThreads2 = 512;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// TMA bulk copies (cp.async.bulk, no LSU work) completing on an mbarrier.
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
// one lane: dst/src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    mbar_expect_tx(bar, bytes);  // before the copy that completes it (tx count never negative)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Issue the window copies of one K2 tile (all warps; warp per window).  The
// warp's window records are fetched with one load per lane up front and
// broadcast with shuffles, so no descriptor load sits on the issue path.
// srec != 0: the tile's records were copied to shared memory (k2_pair_pipe,
// which issues the same tile's windows once per slot), each warp's own
// entries only -- a shared load instead of a global one per slot.
template <class Acc, int NT = kThreads2>
__device__ __forceinline__ void issue_windows(const PassDev& ps, const PassTileDev& tile, const Acc* __restrict__ in,
                                              uint32_t stage, int L, int S, int s0, int H, int ld, int warp,
                                              int lane, uint32_t bar, uint32_t srec = 0u) {
    constexpr int kW = NT / 32;
    for (int base = 0; base < tile.load_cnt; base += 32 * kW) {
        const int mine = base + warp + kW * lane;
        const int4 rec = mine < tile.load_cnt ? (srec ? lds4u(srec + 16u * mine) : ps.loads[tile.load_beg + mine])
                                              : make_int4(0, 0, 0, 0);
        const int cnt = min(32, (tile.load_cnt - base - warp + kW - 1) / kW);
        for (int j = 0; j < cnt; ++j) {
            int4 w;
            w.x = __shfl_sync(0xffffffffu, rec.x, j);
            w.y = __shfl_sync(0xffffffffu, rec.y, j);
            w.z = __shfl_sync(0xffffffffu, rec.z, j);
            w.w = __shfl_sync(0xffffffffu, rec.w, j);
            const Acc* col = in + (size_t)w.x * ld;
            const uint32_t d = stage + static_cast<uint32_t>(w.y) * L * 4u;
            const int start = wrap_any(s0 + w.z, H), n = S + w.w;
            // common case: an aligned window that does not wrap -- whole
            // 16-byte chunks, the last one rounded up (the <= 3 extra words
            // land in the slot's slack; the read stays inside the column's ld)
            const int n4 = (n + 3) & ~3;
            if (!bar && (start & 3) == 0 && start + n <= H && start + n4 <= ld) {
                const Acc* g = col + start + 4 * lane;
                uint32_t sd = d + 16u * lane;
                for (int k = lane; k < (n4 >> 2); k += 32, g += 128, sd += 512u) cp_async16(sd, g);
                continue;
            }
            // rows [start, H) then (past the wrap point) [0, n - (H - start)):
            // 16-byte copies while both sides are 16-byte aligned, 4-byte after
            const int na = min(n, H - start);
            const int run = (start & 3) ? 0 : (na & ~3);
            // copy loops advance a global pointer and a shared offset (no
            // per-copy 64-bit index arithmetic), two copies per iteration
            if (bar) {  // aligned runs by the TMA engine, the rest 4-byte
                if (lane == 0 && run > 0) bulk_copy(d, col + start, run * 4u, bar);
            } else {
                const Acc* g = col + start + 4 * lane;
                uint32_t sd = d + 16u * lane;
                int k = lane;
                for (; 4 * (k + 32) < run; k += 64, g += 256, sd += 1024u) {
                    cp_async16(sd, g);
                    cp_async16(sd + 512u, g + 128);
                }
                if (4 * k < run) cp_async16(sd, g);
            }
            {
                const Acc* g = col + start + run + lane;
                uint32_t sd = d + 4u * (run + lane);
                int i = run + lane;
                for (; i + 32 < na; i += 64, g += 64, sd += 256u) {
                    cp_async4(sd, g);
                    cp_async4(sd + 128u, g + 32);
                }
                if (i < na) cp_async4(sd, g);
            }
            if (n - na <= H) {
                int i0 = na;  // rows past the wrap point: col[i - na]
                if (bar && (na & 3) == 0) {
                    const int nb = (n - na) & ~3;
                    if (lane == 0 && nb > 0) bulk_copy(d + 4u * na, col, nb * 4u, bar);
                    i0 += nb;
                }
                const Acc* g = col + (i0 - na) + lane;
                uint32_t sd = d + 4u * (i0 + lane);
                int i = i0 + lane;
                for (; i + 32 < n; i += 64, g += 64, sd += 256u) {
                    cp_async4(sd, g);
                    cp_async4(sd + 128u, g + 32);
                }
                if (i < n) cp_async4(sd, g);
            } else {  // a window longer than the column (tiny H): wraps again
                for (int i = na + lane; i < n; i += 32) cp_async4(d + 4u * i, col + wrap_any(i - na, H));
            }
        }
    }
}


// TMA windows for k2_pass (PassDev::ktma): the device form of capi.cu
// window_copy for the row tile at s0 -- each window placed at word `delta`
// of its slot so that its long piece is one 16-byte aligned bulk copy; the
// rest by 4-byte cp.async.  The residues go to two 64-bit shared masks (2
// bits per window); the ops add them to the terms that read a window.
__device__ __forceinline__ void issue_windows_dyn(const PassDev& ps, const PassTileDev& tile, const int* __restrict__ in,
                                                  uint32_t stage, int L, int S, int s0, int H, int ld, int warp,
                                                  int lane, uint32_t bar, unsigned long long* smask) {
    constexpr int kW = kThreads2 / 32;
    for (int w = warp; w < tile.load_cnt; w += kW) {
        const int4 l = ps.loads[tile.load_beg + w];  // gcol, slot (= w), off, ext
        const int* __restrict__ col = in + (size_t)l.x * ld;
        const uint32_t d = stage + static_cast<uint32_t>(l.y) * L * 4u;
        const int start = wrap_any(s0 + l.z, H), n = S + l.w;
        int delta, bsrc = 0, bdst = 0, bw = 0, ssrc = 0, sdst = 0, sn = 0;
        if (start + n <= H) {
            delta = start & 3;
            bsrc = start - delta;
            bw = (n + delta + 3) & ~3;
        } else {
            const int a = H - start, b = n - a, c1 = max(0, (H & ~3) - start);
            if (n - c1 <= a) {
                delta = start & 3;
                if (c1 > 0) bsrc = start - delta, bw = c1 + delta;
                ssrc = start + c1, sdst = delta + c1, sn = n - c1;
            } else {
                delta = (4 - (a & 3)) & 3;
                bdst = delta + a, bw = (b + 3) & ~3;
                ssrc = start, sdst = delta, sn = a;
            }
        }
        if (lane == 0) {
            if (bw > 0) bulk_copy(d + 4u * bdst, col + bsrc, 4u * bw, bar);
            if (delta) atomicOr(smask + (w >> 5), static_cast<unsigned long long>(delta) << (2 * (w & 31)));
        }
        uint32_t dd = d + 4u * (sdst + lane);
        int sw = ssrc + lane;
        for (int i = lane; i < sn; i += 32, dd += 128u, sw += 32) cp_async4(dd, col + (sw >= H ? sw - H : sw));
    }
}

// MODE 0: one level per step, 4 rows per lane; 1: rows interleaved over
// lanes; 2: level-pair programs (4-byte accumulators only); 4: level pairs of
// a non-root band, its last step storing the band's columns from registers.
// Root store, reference layout, 4-byte accumulators: rows [0, rows) of the
// tile's columns (slots at sa0 for lanes < 32, sa1 for 32..63) to output
// rows r0.. of slopes t0 + lane; lane = slope, 16-byte shared reads of 4
// rows, 4 coalesced row stores; one row pointer per warp advanced by a fixed
// stride (the 64-bit address math per store dominated otherwise).
template <class Acc, class Out, int NWARPS>
__device__ __forceinline__ void store_root_rows(Out* __restrict__ o, int W, int t0, int nc, uint32_t sa0,
                                                uint32_t sa1, int r0, int rows, int warp, int lane) {
    const size_t wstep = (size_t)W * (NWARPS * 4);
    Out* __restrict__ prow = o + (size_t)(r0 + warp * 4) * W + t0 + lane;
    int i = warp * 4;
    for (; i + 4 <= rows; i += NWARPS * 4, prow += wstep) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (lane + 32 * h >= nc) continue;
            const int4 v4 = lds4u((h ? sa1 : sa0) + i * 4u);
            Out* __restrict__ p = prow + 32 * h;
            p[0] = static_cast<Out>(from_bits<Acc>(v4.x));
            p[W] = static_cast<Out>(from_bits<Acc>(v4.y));
            p[2 * W] = static_cast<Out>(from_bits<Acc>(v4.z));
            p[3 * W] = static_cast<Out>(from_bits<Acc>(v4.w));
        }
    }
    if (i < rows) {  // the last 1-3 rows
        const int nr = rows - i;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (lane + 32 * h >= nc) continue;
            const int4 v4 = lds4u((h ? sa1 : sa0) + i * 4u);
            const int vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < nr) prow[32 * h + (size_t)k * W] = static_cast<Out>(from_bits<Acc>(vv[k]));
        }
    }
}

// The same for tiles of at most 16 slopes: half-warps on two 4-row groups,
// so every lane stores (a 16-slope tile otherwise idles half the warp).
template <class Acc, class Out, int NWARPS>
__device__ __forceinline__ void store_root_rows16(Out* __restrict__ o, int W, int t0, int nc, uint32_t sa, int r0,
                                                  int rows, int warp, int lane) {
    const int sub = lane >> 4, tl = lane & 15;
    const size_t wstep = (size_t)W * (NWARPS * 8);
    Out* __restrict__ prow = o + (size_t)(r0 + warp * 8 + sub * 4) * W + t0 + tl;
    const uint32_t sl = sa + sub * 16u;
    int i = warp * 8;
    if (tl < nc) {
        for (; i + 8 <= rows; i += NWARPS * 8, prow += wstep) {
            const int4 v4 = lds4u(sl + i * 4u);
            prow[0] = static_cast<Out>(from_bits<Acc>(v4.x));
            prow[W] = static_cast<Out>(from_bits<Acc>(v4.y));
            prow[2 * W] = static_cast<Out>(from_bits<Acc>(v4.z));
            prow[3 * W] = static_cast<Out>(from_bits<Acc>(v4.w));
        }
        if (i < rows) {  // the last 1-7 rows
            const int nr = rows - i - sub * 4;
            if (nr > 0) {
                const int4 v4 = lds4u(sl + i * 4u);
                const int vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < nr) prow[(size_t)k * W] = static_cast<Out>(from_bits<Acc>(vv[k]));
            }
        }
    }
}

template <class Acc, class Out, int MODE, bool TMAW = false>
__global__ void __launch_bounds__(kThreads2, 2) k2_pass(PassDev ps, const Acc* __restrict__ src,
                                                     Acc* __restrict__ dst, long long slot_elems, int W, int H,
                                                     int ld, bool final_pass, OutDesc out, QuadSet qs, int img0,
                                                     int pmD) {
    grid_dep_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* sm = reinterpret_cast<Acc*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kWarps = kThreads2 / 32;
    const PassTileDev tile = ps.tiles[blockIdx.y];
    const int S = ps.S, L = ps.L;
    const int s0 = blockIdx.x * S;
    const int slot = blockIdx.z;
    const Acc* __restrict__ in = src + (size_t)slot * slot_elems;

    // 1a. windows of the input columns, 4-byte types: cp.async, every window
    // copy of the tile in flight at once, no register staging (16-byte copies
    // before the wrap point, 4-byte after); issued first so that the op
    // staging below overlaps their flight.  The bulk-copy mbarrier sits in
    // the gap after the slots; one arrival per warp.
    const uint32_t bar = (sizeof(Acc) == 4 && (ps.bulk || TMAW)) ? smem_u32(sm + (size_t)ps.max_slots * L + 8) : 0u;
    // TMAW: the windows' alignment residues, two 64-bit masks after the mbarrier
    unsigned long long* smask = reinterpret_cast<unsigned long long*>(sm + (size_t)ps.max_slots * L + 10);
    if constexpr (sizeof(Acc) == 4) {
        if (bar) {
            if (tid == 0) {
                mbar_init(bar, kWarps);
                smask[0] = 0ull;
                smask[1] = 0ull;
            }
            __syncthreads();
        }
        if constexpr (TMAW) {
            issue_windows_dyn(ps, tile, reinterpret_cast<const int*>(in), smem_u32(sm), L, S, s0, H, ld, warp, lane,
                              bar, smask);
        } else {
            issue_windows<Acc>(ps, tile, in, smem_u32(sm), L, S, s0, H, ld, warp, lane, bar);
        }
        cp_async_commit();
        if (bar) {
            __syncwarp();
            if (lane == 0) mbar_arrive(bar);
        }
    }
    // 0. stage the tile's merge ops in shared memory (after the slots)
    PassOpDev* sops = reinterpret_cast<PassOpDev*>(sm + (size_t)ps.max_slots * L + 16);
    int4* sbops = reinterpret_cast<int4*>(sops);
    int* ssteps = reinterpret_cast<int*>(sops + ps.max_tile_ops);  // the tile's step offsets (after the ops)
    if (tid <= tile.nsteps) ssteps[tid] = ps.step_offs[tile.step_beg + tid];
    const int op0 = ps.step_offs[tile.step_beg], nops = ps.step_offs[tile.step_beg + tile.nsteps] - op0;
    int* swsl = ssteps + 64;  // TMAW: per op, the window each term reads
    if constexpr (MODE == 2 || MODE == 4 || MODE == 6) {
        for (int k = tid; k < 2 * nops; k += kThreads2) sbops[k] = ps.bops[2 * op0 + k];
        if constexpr (TMAW)
            for (int k = tid; k < nops; k += kThreads2) swsl[k] = ps.kwslots[op0 + k];
    } else if constexpr (sizeof(Acc) == 4) {
        for (int k = tid; k < nops; k += kThreads2) sbops[k] = ps.bops[op0 + k];
    } else {
        for (int k = tid; k < nops * 2; k += kThreads2)
            reinterpret_cast<int4*>(sops)[k] = reinterpret_cast<const int4*>(ps.ops + op0)[k];
    }
    // 1b. the windows land (4-byte types) / are loaded through registers (8-byte)
    if constexpr (sizeof(Acc) == 4) {
        cp_async_wait0();
        if (bar) mbar_wait(bar, 0);
    } else {
        for (int l = warp; l < tile.load_cnt; l += kWarps) {
            const int4 ld4 = ps.loads[tile.load_beg + l];
            warp_load_window_v(sm + (size_t)ld4.y * L, in + (size_t)ld4.x * ld, wrap_any(s0 + ld4.z, H), S + ld4.w,
                               H, lane);
        }
    }
    // 2. merge levels
    const uint32_t sbase = smem_u32(sm);
    unsigned long long m0 = 0, m1 = 0;  // TMAW: the windows' residues (read after the first barrier)
    for (int k = 0; k < tile.nsteps; ++k) {
        __syncthreads();
        if constexpr (TMAW) {
            if (k == 0) m0 = smask[0], m1 = smask[1];
        }
        const int ob = ssteps[k] - op0, oe = ssteps[k + 1] - op0;
        if constexpr (MODE == 2 && sizeof(Acc) == 8) {
            run_step_terms64<kWarps, false>(sbase, sbops, ob, oe, warp, lane);
        } else if constexpr (MODE == 4 && sizeof(Acc) == 8) {
            const bool direct = k + 1 == tile.nsteps;
            run_step_terms64<kWarps, true>(sbase, sbops, ob, oe, warp, lane,
                                           direct ? reinterpret_cast<long long*>(dst) + (size_t)slot * slot_elems + s0
                                                  : nullptr,
                                           ld, min(S, H - s0));
        } else if constexpr (MODE == 2) {
            run_step_terms<Acc, kWarps, false, TMAW>(sbase, sbops, ob, oe, warp, lane, nullptr, 0, 0, swsl, m0, m1);
        } else if constexpr (MODE == 6) {
            // u16 pair mode: the root step widens the packed halves to 32 bits
            if (k + 1 < tile.nsteps) run_step_terms<Acc, kWarps, false>(sbase, sbops, ob, oe, warp, lane);
            else run_step_widen<kWarps>(sbase, sbops, ob, oe, warp, lane);
        } else if constexpr (MODE == 4) {
            // the last step of a non-root band stores its columns from registers
            const bool direct = k + 1 == tile.nsteps;
            run_step_terms<Acc, kWarps, true, TMAW>(sbase, sbops, ob, oe, warp, lane,
                                                    direct ? dst + (size_t)slot * slot_elems + s0 : nullptr, ld,
                                                    min(S, H - s0), swsl, m0, m1);
        }
        else if constexpr (sizeof(Acc) == 4)
            run_step_baked<Acc, kWarps, MODE == 1>(sbase, sbops, ob, oe, warp, lane);
        else
            run_step<Acc, kWarps>(sm, L, sops, ob, oe, S, warp, lane);
    }
    __syncthreads();
    // 3. store the tile's columns (window offset 0, rows [s0, s0 + S) clipped to H)
    // (u16 pair mode: the tiles cover words [0, D); word j holds rows j and j + D)
    const int rows = MODE == 6 ? min(S, pmD - s0) : min(S, H - s0);
    const int rows_hi = MODE == 6 ? max(0, min(rows, H - pmD - s0)) : 0;
    if (MODE == 4 && tile.nsteps > 0) return;  // stored by the last step
    if (!final_pass) {
        Acc* __restrict__ o = dst + (size_t)slot * slot_elems;
        const bool al = ((ld | s0) & 3) == 0;
        if constexpr (TMAW) {
            if (tile.nsteps == 0) m0 = smask[0], m1 = smask[1];
        }
        for (int cb = 0; cb < tile.store_cnt; cb += 32 * kWarps) {
            const int mine = cb + warp + kWarps * lane;
            const int2 rec = mine < tile.store_cnt ? (TMAW ? ps.kwstores : ps.stores)[tile.store_beg + mine]
                                                   : make_int2(0, 0);
            const int cnt = min(32, (tile.store_cnt - cb - warp + kWarps - 1) / kWarps);
            for (int j = 0; j < cnt; ++j) {
                const int sl = __shfl_sync(0xffffffffu, rec.x, j);
                int gc = __shfl_sync(0xffffffffu, rec.y, j);
                const Acc* sv = sm + (size_t)sl * L;
                if constexpr (TMAW) {  // a stored window (copy tile): at its alignment residue
                    if (gc & (1 << 30)) {
                        gc &= ~(1 << 30);
                        sv += win_adj(m0, m1, static_cast<unsigned>(sl)) >> 2;
                    }
                }
                // (a shifted window start is not 16-byte aligned: the store takes its scalar path)
                warp_store_col<Acc, Acc>(o + (size_t)gc * ld + s0, sv, rows, al && (sv - sm) % 4 == 0, lane);
            }
        }
    } else {
        const int nq = qs.n;
        int img_l, qi;
        split_slot(slot, nq, img_l, qi);
        Out* __restrict__ o =
            reinterpret_cast<Out*>(out_ptr(out, quad_code(qs, qi))) + (size_t)(img0 + img_l) * out.img_stride;
        const int nc = tile.store_cnt;
        if (out.layout == 0) {
            // the stores of a tile are consecutive slopes: each warp writes rows
            // of nc (<= 64) contiguous t
            const int t0 = ps.stores[tile.store_beg].y;
            const int x0r = lane < nc ? ps.stores[tile.store_beg + lane].x : 0;
            const int x1r = lane + 32 < nc ? ps.stores[tile.store_beg + lane + 32].x : 0;
            // u16 pair mode: .x = lo slot | hi slot << 16
            const int sl0 = MODE == 6 ? (x0r & 0xffff) : x0r, sl1 = MODE == 6 ? (x1r & 0xffff) : x1r;
            if constexpr (sizeof(Acc) == 4) {
                // u16 pair mode: then the upper rows [D + s0, ...) from the hi slots
#pragma unroll 1
                for (int half = 0; half < (MODE == 6 ? 2 : 1); ++half) {
                    const int a0 = half ? x0r >> 16 : sl0, a1 = half ? x1r >> 16 : sl1;
                    const int r0 = half ? s0 + pmD : s0, nr = half ? rows_hi : rows;
                    if (nc <= 16) {  // lane l reads the slot of slope l & 15
                        const int xs = __shfl_sync(0xffffffffu, half ? x0r >> 16 : sl0, lane & 15);
                        store_root_rows16<Acc, Out, kWarps>(o, W, t0, nc, smem_u32(sm + (size_t)xs * L), r0, nr,
                                                            warp, lane);
                    } else {
                        store_root_rows<Acc, Out, kWarps>(o, W, t0, nc, smem_u32(sm + (size_t)a0 * L),
                                                          smem_u32(sm + (size_t)a1 * L), r0, nr, warp, lane);
                    }
                }
            } else {
                for (int i = warp; i < rows; i += kWarps) {
                    Out* __restrict__ orow = o + (size_t)(s0 + i) * W + t0;
                    if (lane < nc) orow[lane] = static_cast<Out>(sm[(size_t)sl0 * L + i]);
                    if (lane + 32 < nc) orow[lane + 32] = static_cast<Out>(sm[(size_t)sl1 * L + i]);
                }
            }
        } else {
            Out* __restrict__ pr = static_cast<Out*>(out.peer);
            if constexpr (MODE == 6) {  // u16 pair mode, slope-major output: both halves
                for (int c = warp; c < nc; c += kWarps) {
                    const int2 st = ps.stores[tile.store_beg + c];
                    const Acc* sv = sm + (size_t)(st.x & 0xffff) * L;
                    const Acc* sh = sm + (size_t)(st.x >> 16) * L;
                    Out* __restrict__ dcol = o + (size_t)st.y * H + s0;
                    for (int i = lane; i < rows; i += 32) dcol[i] = static_cast<Out>(sv[i]);
                    for (int i = lane; i < rows_hi; i += 32) dcol[pmD + i] = static_cast<Out>(sh[i]);
                }
                return;
            }
            for (int c = warp; c < nc; c += kWarps) {
                const int2 st = ps.stores[tile.store_beg + c];
                const Acc* sv = sm + (size_t)st.x * L;
                Out* __restrict__ dcol = o + (size_t)st.y * H + s0;
                if (pr != nullptr && st.y >= out.peer_c0 && st.y < out.peer_c1) {
                    // a slope the other side of the root split needs: also
                    // stored straight into its buffer (peer memory over NVLink)
                    Out* __restrict__ pcol = pr + (size_t)(st.y - out.peer_c0) * H + s0;
                    for (int i = lane; i < rows; i += 32) {
                        const Out v = static_cast<Out>(sv[i]);
                        dcol[i] = v;
                        pcol[i] = v;
                    }
                    continue;
                }
                for (int i = lane; i < rows; i += 32) dcol[i] = static_cast<Out>(sv[i]);
            }
        }
    }
}

// The TMA form of issue_windows for k2_pair_pipe (ps.tma): each window is one
// 16-byte aligned bulk copy by the TMA engine (lane 0 of the warp that owns
// it) plus at most one short run of 4-byte cp.async (the lanes) -- see
// capi.cu window_copy.  Completion: the bulk bytes as mbarrier tx, the
// 4-byte copies through every thread's cp.async.mbarrier.arrive.noinc (the
// barrier counts all kThreads2 threads, so it cannot complete before every
// expect_tx of the slot has been issued).
template <int NT = kThreads2>
__device__ __forceinline__ void issue_windows_tma(uint32_t srec, int nwin, const int* __restrict__ in, int ld,
                                                  uint32_t stage, int H, int warp, int lane, uint32_t bar) {
    constexpr int kW = NT / 32;
    for (int w = warp; w < nwin; w += kW) {
        const int4 r0 = lds4u(srec + 32u * w), r1 = lds4u(srec + 32u * w + 16u);
        const int* __restrict__ col = in + (size_t)r0.x * ld;
        if (lane == 0 && r0.w > 0) bulk_copy(stage + static_cast<uint32_t>(r0.y), col + r0.z, 4u * r0.w, bar);
        uint32_t d = stage + static_cast<uint32_t>(r1.x) + 4u * lane;
        int sw = r1.y + lane;
        for (int i = lane; i < r1.z; i += 32, d += 128u, sw += 32) cp_async4(d, col + (sw >= H ? sw - H : sw));
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// issue_windows_tma on the warps [w0, nw) only (window w -> warp w0 + w mod
// (nw - w0)); no arrival -- every thread arrives separately (tma_arrive).
__device__ __forceinline__ void issue_windows_tma_on(uint32_t srec, int nwin, const int* __restrict__ in, int ld,
                                                     uint32_t stage, int H, int warp, int lane, uint32_t bar, int w0,
                                                     int nw) {
    if (warp < w0) return;
    for (int w = warp - w0; w < nwin; w += nw - w0) {
        const int4 r0 = lds4u(srec + 32u * w), r1 = lds4u(srec + 32u * w + 16u);
        const int* __restrict__ col = in + (size_t)r0.x * ld;
        if (lane == 0 && r0.w > 0) bulk_copy(stage + static_cast<uint32_t>(r0.y), col + r0.z, 4u * r0.w, bar);
        uint32_t d = stage + static_cast<uint32_t>(r1.x) + 4u * lane;
        int sw = r1.y + lane;
        for (int i = lane; i < r1.z; i += 32, d += 128u, sw += 32) cp_async4(d, col + (sw >= H ? sw - H : sw));
    }
}
__device__ __forceinline__ void tma_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// ------------------------------------------------------- K2, pair mode
// The u16 pair mode root band with double-buffered windows: each CTA keeps
// its tile and walks slots (grid.z strided).  While slot i computes, the
// windows of slot i + 1 stream into the second buffer (load-space slots
// moved by ps.pipe_delta; the op and store tables carry both variants), so
// the copies' latency hides behind the merges.  Tiles of <= 16 slopes,
// reference layout only (the launcher falls back to k2_pass MODE 6).
// WIDE: tiles of 17..32 slopes on 1024 threads, one CTA per SM (the two
// window buffers of a 32-slope tile take ~175 KB): half the root store's
// partial-line writes and fewer windows per slope than 16-slope tiles.
// PROBE: compiled with the FHT_K2_PROBE timing switches (PassDev::probe)
template <class Out, bool TMA, bool WIDE = false, bool PROBE = false>
__global__ void __launch_bounds__(WIDE ? 1024 : kThreads2, WIDE ? 1 : 2)
    k2_pair_pipe(PassDev ps, const int* __restrict__ src, long long slot_elems, int W, int H, int ld, OutDesc out,
                 QuadSet qs, int img0, int pmD, int nslots) {
    using Acc = int;
    constexpr int kNT = WIDE ? 1024 : kThreads2;
    constexpr int kWarps = kNT / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* sm = reinterpret_cast<Acc*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const PassTileDev tile = ps.tiles[blockIdx.y];
    const int S = ps.S, L = ps.L;
    const int s0 = blockIdx.x * S;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t alt = static_cast<uint32_t>(ps.pipe_delta) * static_cast<uint32_t>(L) * 4u;
    int slot = blockIdx.z;
    // the tile's op tables (both buffers) and step offsets, then the first
    // slot's windows (those wait for the previous kernel)
    int4* sbops = reinterpret_cast<int4*>(sm + (size_t)(ps.pipe_delta + ps.pipe_loads) * L + 16);
    const int op0 = ps.step_offs[tile.step_beg], nops = ps.step_offs[tile.step_beg + tile.nsteps] - op0;
    int* ssteps = reinterpret_cast<int*>(sbops + 4 * ps.max_tile_ops);
    if (tid <= tile.nsteps) ssteps[tid] = ps.step_offs[tile.step_beg + tid] - op0;
    const bool oq_fixed = static_cast<int>(gridDim.z) % qs.n == 0;
    Out* __restrict__ oq = nullptr;  // (oq_fixed) the CTA's quadrant output, at image img0
    if (oq_fixed) {
        int img_l, qi;
        split_slot(slot, qs.n, img_l, qi);
        oq = reinterpret_cast<Out*>(out_ptr(out, quad_code(qs, qi))) + (size_t)img0 * out.img_stride;
    }
    const int so1 = tile.nsteps >= 1 ? ps.step_offs[tile.step_beg + 1] - op0 : 0;
    const int so2 = tile.nsteps >= 2 ? ps.step_offs[tile.step_beg + 2] - op0 : 0;
    const uint32_t sops0 = smem_u32(sbops);
    {
        const int4* __restrict__ b0 = TMA ? ps.tbops : ps.bops;
        const int4* __restrict__ b1 = TMA ? ps.tbops1 : ps.bops1;
        for (int k = tid; k < 2 * nops; k += kNT) {
            sbops[k] = b0[2 * op0 + k];
            sbops[2 * nops + k] = b1[2 * op0 + k];
        }
    }
    const int nc = tile.store_cnt;
    const int t0 = ps.stores[tile.store_beg].y;
    const int sl = WIDE ? lane : (lane & 15);  // the slope whose root slots this lane stores
    const int xs0 = sl < nc ? ps.stores[tile.store_beg + sl].x : 0;
    const int xs1 = sl < nc ? ps.stores1[tile.store_beg + sl].x : 0;
    const int rows = min(S, pmD - s0), rows_hi = max(0, min(rows, H - pmD - s0));
    // the window records, after the step offsets: each warp copies the
    // entries it will issue (so a __syncwarp orders them)
    const uint32_t srec = smem_u32(ssteps + 64);
    // TMA: two window records per load, then the two buffers' mbarriers
    const uint32_t bars = srec + (TMA ? 32u : 16u) * static_cast<uint32_t>(ps.pipe_loads);
    if constexpr (TMA) {
        for (int k = warp; k < tile.load_cnt; k += kWarps)  // each warp stages the records it will issue
            if (lane < 2) sts4u(srec + 32u * k + 16u * lane, ps.twin[2 * tile.load_beg + 2 * k + lane]);
        if (tid == 0) {
            mbar_init(bars, kNT);
            mbar_init(bars + 8u, kNT);
        }
        __syncthreads();
    } else {
        for (int mine = warp + kWarps * lane; mine < tile.load_cnt; mine += 32 * kWarps)
            sts4u(srec + 16u * mine, ps.loads[tile.load_beg + mine]);
        __syncwarp();
    }
    grid_dep_wait();
    if constexpr (TMA) {
        issue_windows_tma<kNT>(srec, tile.load_cnt, src + (size_t)slot * slot_elems, ld, sbase, H, warp, lane, bars);
    } else {
        issue_windows<Acc, kNT>(ps, tile, src + (size_t)slot * slot_elems, sbase, L, S, s0, H, ld, warp, lane, 0u, srec);
        cp_async_commit();
    }
    const int probe = PROBE ? ps.probe : 0;
    for (int it = 0;; ++it) {
        const int p = it & 1;
        if (it == 0 || !(probe & 4)) {
            if constexpr (TMA) {
                mbar_wait(bars + 8u * p, (it >> 1) & 1);  // this slot's windows (bulk bytes + 4-byte copies)
            } else {
                cp_async_wait0();  // this slot's windows
            }
        }
        __syncthreads();   // ... visible to all; the last slot's store is done with the other buffer
        const int next = slot + static_cast<int>(gridDim.z);
        // (TMA, two steps: the next slot's windows are issued after step 0,
        // by the warps that have one op fewer in it -- they would wait at the
        // step barrier anyway -- so no warp starts its first op late)
        const bool defer = TMA && !WIDE && tile.nsteps == 2;
        if (next < nslots && !(probe & 4) && !defer) {
            if constexpr (TMA) {
                // the other buffer was last read (and some of its slots
                // written) through the generic proxy before the barrier above
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_windows_tma<kNT>(srec, tile.load_cnt, src + (size_t)next * slot_elems, ld, sbase + (p ? 0u : alt), H,
                                  warp, lane, bars + 8u * (1 - p));
            } else {
                issue_windows<Acc, kNT>(ps, tile, src + (size_t)next * slot_elems, sbase + (p ? 0u : alt), L, S, s0, H,
                                        ld, warp, lane, 0u, srec);
                cp_async_commit();
            }
        }
        const uint32_t ops = sops0 + (p ? 32u * static_cast<uint32_t>(nops) : 0u);
        // the op ranges of the first two steps (all of a root band of <= 4
        // levels) come from registers, not from the shared step table
        for (int k = 0; k < ((probe & 1) ? 0 : tile.nsteps); ++k) {
            if (k) {
                if constexpr (TMA && !WIDE) {
                    if (defer && k == 1 && next < nslots && !(probe & 4)) {
                        // warps [so1 - kWarps, kWarps) ran one op fewer in step 0 (all warps when so1 <= kWarps)
                        const int w0 = so1 > kWarps ? min(so1 - kWarps, kWarps - 1) : 0;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue_windows_tma_on(srec, tile.load_cnt, src + (size_t)next * slot_elems, ld,
                                             sbase + (p ? 0u : alt), H, warp, lane, bars + 8u * (1 - p), w0, kWarps);
                        tma_arrive(bars + 8u * (1 - p));
                    }
                }
                __syncthreads();
            }
            const int lo = k == 0 ? 0 : k == 1 ? so1 : ssteps[k];
            const int hi = k == 0 ? so1 : k == 1 ? so2 : ssteps[k + 1];
            if (k + 1 < tile.nsteps) {
                run_step_terms_s<kWarps>(sbase, ops, lo, hi, warp, lane);
            } else {
                run_step_widen_s<kWarps>(sbase, ops, lo, hi, warp, lane);
            }
        }
        __syncthreads();
        // this slot's output image: the quadrant is the same for every slot of
        // the CTA when the slot stride is a multiple of the quadrant count
        Out* __restrict__ o;
        if (oq_fixed) {
            int img_l, qi;
            split_slot(slot, qs.n, img_l, qi);
            o = oq + (size_t)img_l * out.img_stride;
        } else {
            int img_l, qi;
            split_slot(slot, qs.n, img_l, qi);
            o = reinterpret_cast<Out*>(out_ptr(out, quad_code(qs, qi))) + (size_t)(img0 + img_l) * out.img_stride;
        }
        const int xs = p ? xs1 : xs0;
        if (probe & 2) {
        } else if constexpr (WIDE) {
            store_root_rows<Acc, Out, kWarps>(o, W, t0, nc, sbase + static_cast<uint32_t>(xs & 0xffff) * L * 4u, 0u, s0,
                                              rows, warp, lane);
            if (rows_hi > 0)
                store_root_rows<Acc, Out, kWarps>(o, W, t0, nc, sbase + static_cast<uint32_t>(xs >> 16) * L * 4u, 0u,
                                                  s0 + pmD, rows_hi, warp, lane);
        } else {
            store_root_rows16<Acc, Out, kWarps>(o, W, t0, nc, sbase + static_cast<uint32_t>(xs & 0xffff) * L * 4u, s0,
                                                rows, warp, lane);
            if (rows_hi > 0)
                store_root_rows16<Acc, Out, kWarps>(o, W, t0, nc, sbase + static_cast<uint32_t>(xs >> 16) * L * 4u,
                                                    s0 + pmD, rows_hi, warp, lane);
        }
        slot = next;
        if (slot >= nslots) break;
    }
}

// ------------------------------------------------------------ root merge
// The root level from its two children held as separate slope-major column
// ranges (the multi-GPU root split): output slopes [t_beg,
// t_end) of a width-W node, OUT[t][s] = L[t0][s] + R[t1][(s + r) mod H]
// (transform.cpp:46-57), tiles of 32 slopes x 32 shifts transposed through
// shared memory into the reference layout (or written slope-major).
template <class Acc, class Out>
__global__ void __launch_bounds__(256) k_merge_root(const int4* __restrict__ ops, const Acc* __restrict__ left,
                                                     int left_first, const Acc* __restrict__ right, int right_first,
                                                     int W, int H, int t_beg, int t_end, Out* __restrict__ out,
                                                     int layout) {
    __shared__ Acc tile[32][33];
    const int lane = threadIdx.x, ty = threadIdx.y;
    const int t0 = t_beg + blockIdx.x * 32, s0 = blockIdx.y * 32;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int tl = ty + 8 * j, t = t0 + tl, s = s0 + lane;
        if (t < t_end && s < H) {
            const int4 op = ops[t];  // (t, t0, t1, r)
            int jb = s + op.w;
            if (jb >= H) jb -= H;
            tile[tl][lane] = left[(size_t)(op.y - left_first) * H + s] + right[(size_t)(op.z - right_first) * H + jb];
        }
    }
    __syncthreads();
    if (layout == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int sl = ty + 8 * j, s = s0 + sl, t = t0 + lane;
            if (s < H && t < t_end) out[(size_t)s * W + t] = static_cast<Out>(tile[lane][sl]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int tl = ty + 8 * j, t = t0 + tl, s = s0 + lane;
            if (t < t_end && s < H) out[(size_t)t * H + s] = static_cast<Out>(tile[tl][lane]);
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
// Opt a kernel into the full 227 KB of dynamic shared memory once per
// (device, kernel) instead of on every launch (host overhead on small images).
void allow_smem(const void* fn) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({dev, fn}).second)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

// Slots one k2_pair_pipe CTA walks: FHT_K2_SLOTS_PER_CTA, else as many as
// keep >= 3 waves of 2 CTAs per SM, at most 8 (measured best for c4: 8 at
// 256 images, 4 at the 32 images of a rank under 8-GPU strong scaling).
int slots_per_cta(int ctas_at_one, int nslots) {
    if (const char* e = std::getenv("FHT_K2_SLOTS_PER_CTA")) return std::max(1, std::min(64, std::atoi(e)));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return std::max(1, std::min({8, nslots, ctas_at_one / (sms * 2 * 3)}));
}

// K1's (pair mode) L2 prefetch distance; FHT_K1_PREFETCH (0: off)
int k1_prefetch_ahead() {
    if (const char* e = std::getenv("FHT_K1_PREFETCH")) return std::max(0, std::atoi(e));
    return 64;
}

// K1P's L2 prefetch distance in CTAs (launch order): about one wave of two
// CTAs per SM; FHT_K1P_PREFETCH overrides it (0: off)
int k1p_prefetch_ahead() {
    if (const char* e = std::getenv("FHT_K1P_PREFETCH")) return std::max(0, std::atoi(e));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 2 * sms;
}

// FHT_K2_PROBE (debug timing only, see PassDev::probe)
int k2_probe() {
    static const int v = [] {
        const char* e = std::getenv("FHT_K2_PROBE");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

template <class In, class Acc, class Out>
int launch_typed(const GroupLaunch& g, cudaStream_t st, LaunchHook hook, void* ctx) {
    int launches = 0;
    const int nslots = g.nimg * g.qs.n;
    const size_t smem = k1_smem_bytes(g.acc_dtype, g.k1_max_width, g.k1_sr, g.k1_max_ops, g.k1_max_steps);
    Acc* ws = reinterpret_cast<Acc*>(g.ws);
    // Pass 0: the width-32 Brady-Yong blocks (K1P) and the other blocks (K1)
    // write disjoint columns; when both exist, K1 runs concurrently on the
    // plan's auxiliary stream (forked after the staging, joined by an event
    // before the first K2 pass).
    // u8 staging (large batches): the aligned working columns K1 and K1P read
    const unsigned char* stage = nullptr;
    if constexpr (sizeof(Acc) == 4 && std::is_same<In, unsigned char>::value) {
        if ((g.nby > 0 || g.pm_D) && g.stage != nullptr) {
            const auto* im = reinterpret_cast<const unsigned char*>(g.img);
            const long long ext_w = std::max<long long>(g.img_w, g.stage_p >= 0 ? g.stage_pitch : 0);
            const long long ext_h = std::max<long long>(g.img_h, g.stage_t >= 0 ? g.stage_pitch : 0);
            dim3 gs(static_cast<unsigned>((ext_w + 63) / 64), static_cast<unsigned>((ext_h + 63) / 64), g.nimg);
            NvtxRange nr("fht: u8 staging");
            launch_k(g.pdl, k_stage_u8, gs, dim3(256), 0, st, im, g.img_w, g.img_h, g.img_pitch, g.img_stride, g.img0,
                     g.stage, g.stage_img, g.stage_pitch, g.stage_t, g.stage_pitch, g.stage_p);
            ++launches;
            if (hook) hook(ctx, 5);
            stage = g.stage;
        }
    }
    const bool both = (sizeof(Acc) == 4) && g.nby > 0 && g.nblocks > 0 && g.aux_stream && g.fork_mu && !hook;
    cudaStream_t st1 = both ? g.aux_stream : st;
    // cudaStreamWaitEvent binds to the event's most recent record at call
    // time, so holding the plan's lock across each record + wait pair is all
    // concurrent callers need (they may then share the aux stream: at worst a
    // false dependency, never a missing one)
    auto fork_join = [&](cudaEvent_t ev, cudaStream_t from, cudaStream_t to) {
        std::lock_guard<std::mutex> lk(*static_cast<std::mutex*>(g.fork_mu));
        cudaEventRecord(ev, from);
        cudaStreamWaitEvent(to, ev, 0);
    };
    if (both) fork_join(g.ev_fork, st, st1);
    bool pass0_done = false;
    if constexpr (sizeof(Acc) == 8 && std::is_same<Acc, long long>::value && !std::is_same<In, unsigned char>::value) {
        if (g.k1_acc32) {
            // pass 0 in int32, block roots widened to int64 on the store
            // (K1 on the main stream after K1P: two short launches)
            if (g.nby > 0) {
                NvtxRange nr("fht: pass 0, width-32 blocks (K1P, int32 -> int64)");
                auto kb = k1_by32<In, int32_t, 5, kThreadsBYP, long long>;
                allow_smem(reinterpret_cast<const void*>(kb));
                dim3 gb((g.H + g.S - 1) / g.S, g.nby, nslots);
                launch_k(g.pdl, kb, gb, dim3(kThreadsBYP), k1_by32_smem_bytes(), st, reinterpret_cast<const In*>(g.img),
                         g.img_w, g.img_h, g.img_pitch, g.img_stride, g.img0, g.qs, g.W, g.H, g.ld, g.S, g.by_x0, ws, g.nbuf,
                         static_cast<const unsigned char*>(nullptr), 0LL, 0LL, -1LL, -1LL, 0);
                ++launches;
                if (hook) hook(ctx, 4);
            }
            if (g.nblocks > 0) {
                NvtxRange nr("fht: pass 0, generic blocks (K1, int32 -> int64)");
                const size_t smem32 = k1_smem_bytes(kI32, g.k1_max_width, g.k1_sr, g.k1_max_ops, g.k1_max_steps);
                dim3 g1((g.H + g.S - 1) / g.S, g.nblocks, nslots);
                auto k1 = k1_blocks<In, int32_t, Out, true, long long>;
                allow_smem(reinterpret_cast<const void*>(k1));
                launch_k(g.pdl, k1, g1, dim3(kThreads), smem32, st, reinterpret_cast<const In*>(g.img), g.img_w,
                         g.img_h, g.img_pitch, g.img_stride, g.img0, g.qs, g.W, g.H, g.ld, g.S, g.blocks, g.shapes,
                         g.step_offs, g.k1_ops, g.k1_bops, g.k1_max_width, g.k1_sr, g.k1_max_ops, ws, g.nbuf,
                         g.root_is_block, g.out, static_cast<const unsigned char*>(nullptr), 0LL, 0LL, -1LL, -1LL, 0,
                         0);
                ++launches;
                if (hook) hook(ctx, 1);
            }
            pass0_done = true;
        }
    }
    if (!pass0_done && g.nblocks > 0) {
        NvtxRange nr("fht: pass 0, generic blocks (K1)");
        dim3 g1(g.pm_D ? 1 : (g.H + g.S - 1) / g.S, g.nblocks, nslots);
        auto k1 = g.k2_scalar && sizeof(Acc) == 4 ? k1_blocks<In, Acc, Out, true> : k1_blocks<In, Acc, Out, false>;
        allow_smem(reinterpret_cast<const void*>(k1));
        launch_k(g.pdl && !both, k1, g1, dim3(kThreads), smem, st1, reinterpret_cast<const In*>(g.img), g.img_w,
                 g.img_h, g.img_pitch, g.img_stride, g.img0, g.qs, g.W, g.H, g.ld, g.S, g.blocks, g.shapes, g.step_offs,
                 g.k1_ops, g.k1_bops, g.k1_max_width, g.k1_sr, g.k1_max_ops, ws, g.nbuf, g.root_is_block, g.out, stage,
                 g.stage_pitch, g.stage_img, g.stage_t, g.stage_p, g.pm_D, k1_prefetch_ahead());
        ++launches;
        if (hook) hook(ctx, 1);
    }
    if constexpr (sizeof(Acc) == 4) {
        if (g.nby > 0) {
            NvtxRange nr("fht: pass 0, width-32 blocks (K1P)");
            auto kb = g.k1p_variant == 0   ? k1_by32<In, Acc, 0>
                      : g.k1p_variant == 2 ? k1_by32<In, Acc, 2>
                      : g.k1p_variant == 3 ? k1_by32<In, Acc, 3>
                      : g.k1p_variant == 4 ? k1_by32<In, Acc, 4>
                                           : k1_by32<In, Acc, 5>;
            const int sm_by = static_cast<int>(k1_by32_smem_bytes());
            bool launched = false;
            if constexpr (std::is_same<In, unsigned char>::value && std::is_same<Acc, int32_t>::value) {
                // the pair mode's K1P: 576 threads (FHT_K1P_PAIR576=0: the 512-thread kernel)
                if (g.pm_D && stage && g.k1p_pair576) {
                    auto kq = k1_by32_pair<Acc>;
                    allow_smem(reinterpret_cast<const void*>(kq));
                    launch_k(g.pdl, kq, dim3(1, g.nby, nslots), dim3(kThreadsBYP), sm_by, st, g.qs, g.W, g.H, g.ld, g.S,
                             g.by_x0, ws, g.nbuf, stage, g.stage_pitch, g.stage_img, g.stage_t, g.stage_p, g.pm_D,
                             k1p_prefetch_ahead());
                    launched = true;
                }
            }
            // variant 5 outside the pair mode: 576 threads (FHT_K1P_576=0: 512)
            const bool t576 = !launched && g.k1p_variant == 5 && g.k1p_576 && !(stage && g.pm_D);
            if (t576) kb = k1_by32<In, Acc, 5, kThreadsBYP>;
            if (!launched) {
                allow_smem(reinterpret_cast<const void*>(kb));
                dim3 gb(g.pm_D ? 1 : (g.H + g.S - 1) / g.S, g.nby, nslots);
                launch_k(g.pdl, kb, gb, dim3(t576 ? kThreadsBYP : kThreadsBY), sm_by, st, reinterpret_cast<const In*>(g.img), g.img_w,
                         g.img_h, g.img_pitch, g.img_stride, g.img0, g.qs, g.W, g.H, g.ld, g.S, g.by_x0, ws, g.nbuf,
                         stage, g.stage_pitch, g.stage_img, g.stage_t, g.stage_p, stage ? g.pm_D : 0);
            }
            ++launches;
            if (hook) hook(ctx, 4);
        }
    }
    if (both) fork_join(g.ev_join, st1, st);
    if (g.root_is_block) return launches;
    const long long slot_elems = (long long)g.nbuf * g.W * g.ld;
    for (int p = 0; p < g.npasses; ++p) {
        const PassDev& ps = g.passes[p];
        const bool final_pass = (p == g.npasses - 1);
        NvtxRange nr(final_pass ? "fht: root band (K2)" : "fht: upper band (K2)");
        const Acc* SRC = ws + (size_t)(p & 1) * g.W * g.ld;          // pass p reads buffer (p-1)%2 ... K1 wrote 0
        Acc* DST = ws + (size_t)((p + 1) & 1) * g.W * g.ld;
        const size_t smem2 = k2_smem_bytes(g.acc_dtype, ps.max_slots, ps.L, ps.max_tile_ops);
        auto k2 = k2_pass<Acc, Out, 0>;
        if constexpr (sizeof(Acc) == 8) {
            // int64: level pairs on 64-bit words; non-root bands store from registers
            if (ps.pairs) k2 = final_pass ? k2_pass<Acc, Out, 2> : k2_pass<Acc, Out, 4>;
        }
        if constexpr (sizeof(Acc) == 4) {
            // level pairs; non-root bands (MODE 4) store their columns from registers
            if (ps.pairs) k2 = final_pass ? k2_pass<Acc, Out, 2> : k2_pass<Acc, Out, 4>;
            else if (g.k2_scalar) k2 = k2_pass<Acc, Out, 1>;
            if constexpr (std::is_same<Acc, int32_t>::value) {
                if (ps.pairs && final_pass && g.pm_D) k2 = k2_pass<Acc, Out, 6>;  // u16 pair mode root band
            }
        }
        PassDev pd = ps;
        pd.bulk = g.k2_bulk;
        pd.probe = k2_probe();
        if constexpr (std::is_same<Acc, int32_t>::value) {
            // pair-mode root band with double-buffered windows
            int max_nc = 0;
            (void)max_nc;
            if (g.pm_D && final_pass && ps.pairs && ps.pipe_delta > 0 && !g.k2_bulk && g.out.layout == 0 &&
                ps.tile_nc_max <= 32) {
                const bool wide = ps.tile_nc_max > 16;
                const bool tma = ps.tma && ps.twin != nullptr;
                const size_t smp = k2_smem_bytes(g.acc_dtype, ps.pipe_delta + ps.pipe_loads, ps.L, 2 * ps.max_tile_ops) +
                                   static_cast<size_t>(ps.pipe_loads) * sizeof(int4) * (tma ? 2 : 1) +  // window records
                                   16;                                                                   // mbarriers
                auto kp = wide ? (tma ? k2_pair_pipe<Out, true, true> : k2_pair_pipe<Out, false, true>)
                          : pd.probe ? (tma ? k2_pair_pipe<Out, true, false, true> : k2_pair_pipe<Out, false, false, true>)
                                     : (tma ? k2_pair_pipe<Out, true> : k2_pair_pipe<Out, false>);
                allow_smem(reinterpret_cast<const void*>(kp));
                const int rt = (g.pm_D + ps.S - 1) / ps.S;
                const int spc = slots_per_cta(rt * ps.ntiles * nslots, nslots);
                dim3 gp(rt, ps.ntiles, (nslots + spc - 1) / spc);
                launch_k(g.pdl, kp, gp, dim3(wide ? 1024 : kThreads2), smp, st, pd, SRC, slot_elems, g.W, g.H, g.ld, g.out, g.qs,
                         g.img0, g.pm_D, nslots);
                ++launches;
                if (hook) hook(ctx, 3);
                continue;
            }
        }
        size_t smem2t = smem2;
        if constexpr (sizeof(Acc) == 4) {
            // level-pair bands (not the pair mode's): windows by the TMA engine
            if (ps.pairs && ps.ktma && !g.pm_D && !g.k2_bulk) {
                k2 = final_pass ? k2_pass<Acc, Out, 2, true> : k2_pass<Acc, Out, 4, true>;
                smem2t += static_cast<size_t>(ps.max_tile_ops) * sizeof(int);  // the ops' window indices
            }
        }
        allow_smem(reinterpret_cast<const void*>(k2));
        dim3 g2(((g.pm_D ? g.pm_D : g.H) + ps.S - 1) / ps.S, ps.ntiles, nslots);
        launch_k(g.pdl, k2, g2, dim3(kThreads2), smem2t, st, pd, SRC, DST, slot_elems, g.W, g.H, g.ld, final_pass, g.out,
                 g.qs, g.img0, g.pm_D);
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
    (void)max_ops;
    (void)max_steps;
    return k1_ops_offset(acc_dtype, max_width, sr) + 64;  // two slot buffers + vector-read slack
}

size_t k2_smem_bytes(int acc_dtype, int max_slots, int L, int max_tile_ops) {
    const size_t esz = acc_dtype == kI64 ? 8 : 4;
    // slots, +16 elements of vector-merge read slack, the staged ops, the step offsets
    return (static_cast<size_t>(max_slots) * L + 16) * esz + static_cast<size_t>(max_tile_ops) * sizeof(PassOpDev) +
           64 * sizeof(int);
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

int launch_merge_root(const int4* d_ops, const void* left, int left_first, const void* right, int right_first,
                      int W, int H, int t_beg, int t_end, void* out, int acc, int outd, int layout, cudaStream_t st) {
    if (t_end <= t_beg) return 0;
    dim3 g((t_end - t_beg + 31) / 32, (H + 31) / 32);
    dim3 b(32, 8);
#define FHT_MERGE(A, O)                                                                                        \
    k_merge_root<A, O><<<g, b, 0, st>>>(d_ops, static_cast<const A*>(left), left_first,                       \
                                        static_cast<const A*>(right), right_first, W, H, t_beg, t_end,          \
                                        static_cast<O*>(out), layout)
    if (acc == kI32 && outd == kI32) FHT_MERGE(int32_t, int32_t);
    else if (acc == kI32 && outd == kI64) FHT_MERGE(int32_t, long long);
    else if (acc == kI64 && outd == kI64) FHT_MERGE(long long, long long);
    else if (acc == kF32 && outd == kF32) FHT_MERGE(float, float);
    else return -1;
#undef FHT_MERGE
    return 1;
}

void launch_absmax(const void* d_in, int dtype, long long n, unsigned long long* d_max, cudaStream_t st) {
    const int blocks = 148 * 4;
    if (dtype == kI32)
        k_absmax<int32_t><<<blocks, 256, 0, st>>>(reinterpret_cast<const int32_t*>(d_in), n, d_max);
    else if (dtype == kI64)
        k_absmax<long long><<<blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(d_in), n, d_max);
}

}  // namespace fhtb
