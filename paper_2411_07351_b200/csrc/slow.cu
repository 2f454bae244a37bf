// slow.cu -- structure-free direct summation on the device, the GPU form of
// the reference's validation oracle slow_hough (oracle.cpp:9-25):
//     J(t, s) = sum_x I(x, (pat_t(x) + s) mod h)
// with pat_t the Algorithm-2 pattern (pattern.cpp:10-30) built on the host.
// Theta(w^2 h) work: it exists to check the fast path at sizes where the CPU
// oracle is infeasible, not for speed.
#include <cuda_runtime.h>

#include <cstdint>

#include "slow.cuh"

namespace fhtb {
namespace {

// The working column-major copy of one quadrant: cols[x*h + y].
template <class In>
__global__ void k_columns(const In* __restrict__ img, int img_w, int img_h, int q, long long* __restrict__ cols,
                          int W, int H) {
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int x = static_cast<int>(k / H), y = static_cast<int>(k % H);
        long long v;
        switch (q) {
            case 0: v = static_cast<long long>(img[(size_t)y * img_w + x]); break;
            case 1: v = static_cast<long long>(img[(size_t)y * img_w + (img_w - 1 - x)]); break;
            case 2: v = static_cast<long long>(img[(size_t)x * img_w + y]); break;
            default: v = static_cast<long long>(img[(size_t)(img_h - 1 - x) * img_w + y]); break;
        }
        cols[k] = v;
    }
}

// One thread per (t, s); lanes over consecutive s read consecutive rows of
// each column (coalesced); the pattern row is warp-uniform.
__global__ void k_slow(const long long* __restrict__ cols, const int* __restrict__ pat, int W, int H,
                       long long* __restrict__ out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (s >= H) return;
    const int* __restrict__ p = pat + (size_t)t * W;
    long long acc = 0;
    for (int x = 0; x < W; ++x) {
        int y = (p[x] % H) + s;
        if (y >= H) y -= H;
        acc += cols[(size_t)x * H + y];
    }
    out[(size_t)s * W + t] = acc;  // reference layout hough[s*W + t]
}

}  // namespace

void launch_slow_hough(const void* img, int in_dtype, int img_w, int img_h, int q, const int* d_pat, int W, int H,
                       long long* d_cols, long long* d_out, cudaStream_t st) {
    const int blocks = 148 * 8;
    if (in_dtype == 0)
        k_columns<uint8_t><<<blocks, 256, 0, st>>>(static_cast<const uint8_t*>(img), img_w, img_h, q, d_cols, W, H);
    else if (in_dtype == 1)
        k_columns<int32_t><<<blocks, 256, 0, st>>>(static_cast<const int32_t*>(img), img_w, img_h, q, d_cols, W, H);
    else
        k_columns<long long><<<blocks, 256, 0, st>>>(static_cast<const long long*>(img), img_w, img_h, q, d_cols, W,
                                                     H);
    dim3 g((H + 255) / 256, W);
    k_slow<<<g, 256, 0, st>>>(d_cols, d_pat, W, H, d_out);
}

}  // namespace fhtb

// ------------------------------------------------------------- analysis
// The paper's accuracy sweep (analysis.cpp:63-91, 231-243) on the device:
// for every width n and slope t, max over x of |x t - pat(n,t)(x) (n-1)|, the
// numerator of the max orthotropic error E(n) = worst / (n-1).  pat(n,t)(x)
// is found by descending Algorithm 2's split tree from the root (pattern.cpp:
// 10-20): O(log n) per point, no tables; unsigned 32-bit products are exact
// for n <= 46340.
namespace fhtb {
namespace {

__device__ __forceinline__ unsigned pattern_value(unsigned n, unsigned t, unsigned x, int strategy) {
    unsigned w = n, x0 = 0, tn = t, lift = 0;
    while (w > 1) {
        const unsigned w0 = strategy == 0 ? (w >> 1) : (1u << (31 - __clz(w - 1)));  // split.hpp:33-44
        const unsigned w1 = w - w0, den2 = 2 * (w - 1);
        if (x < x0 + w0) {
            tn = (2 * tn * (w0 - 1) + (w - 1)) / den2;  // round_half_up_ratio, split.hpp:53-57
            w = w0;
        } else {
            const unsigned t1 = (2 * tn * (w1 - 1) + (w - 1)) / den2;
            lift += tn - t1;
            tn = t1;
            x0 += w0;
            w = w1;
        }
    }
    return lift;
}

// grid: x = chunk of 8 slopes, y = n - n_lo; warp per slope, lanes over x.
__global__ void k_max_deviation(int n_lo, int strategy, unsigned long long* __restrict__ worst) {
    const unsigned n = n_lo + blockIdx.y;
    const unsigned t = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t >= n) return;  // warp-uniform
    const unsigned lane = threadIdx.x & 31;
    unsigned long long m = 0;
    for (unsigned x = lane; x < n; x += 32) {
        const long long d = (long long)x * t - (long long)pattern_value(n, t, x, strategy) * (long long)(n - 1);
        const unsigned long long a = d < 0 ? -d : d;
        m = a > m ? a : m;
    }
    for (int off = 16; off; off >>= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, m, off);
        m = o > m ? o : m;
    }
    if (lane == 0) atomicMax(worst + blockIdx.y, m);
}

}  // namespace

void launch_max_deviation(int n_lo, int n_hi, int strategy, unsigned long long* d_worst, cudaStream_t st) {
    dim3 g((n_hi + 7) / 8, n_hi - n_lo + 1);
    k_max_deviation<<<g, 256, 0, st>>>(n_lo, strategy, d_worst);
}

}  // namespace fhtb
