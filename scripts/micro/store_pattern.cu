// Store-pattern micro-benchmark for the K2 root store (c4: 1024 slots of a
// 509 x 509 int32 Hough image in the reference layout hough[s*W + t]).
// Each variant writes the same 1.06 GB; times are CUDA events, best of 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 store_pattern.cu -o /tmp/sp && /tmp/sp
#include <cstdio>
#include <cuda_runtime.h>

constexpr int H = 509, NSLOT = 1024;
#ifndef PW
#define PW 509
#endif
#ifndef OFF
#define OFF 0
#endif
constexpr int W = 509, RS = PW;  // RS: row stride in ints (512 = line-aligned rows)
constexpr long long SLOT = (long long)RS * H;

// A: plain coalesced write of the whole buffer
__global__ void k_linear(int4* o, long long n4) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        o[i] = make_int4(1, 2, 3, 4);
}

// B: the production pattern -- tile of TW slopes, each CTA walks SPC slots
// (grid.z strided), half-warps (TW = 16) or warps (TW = 32) on row pieces,
// 4 rows per lane per iteration; ROWS_PER_WARP_ITER rows per warp pass
template <int TW>
__global__ void __launch_bounds__(512, 2) k_tiles(int* o, int nslots, int ntiles) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.y, t0 = tile * TW;
    constexpr int G = 32 / TW;  // row groups per warp
    const int sub = lane / TW, tl = lane % TW;
    const int nc = min(TW, W - t0);
    for (int slot = blockIdx.z; slot < nslots; slot += gridDim.z) {
        int* base = o + slot * SLOT + OFF;
        if (tl < nc)
            for (int i = warp * 4 * G + sub * 4; i < H; i += 16 * 4 * G) {
                int* p = base + (long long)i * RS + t0 + tl;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (i + k < H) p[(long long)k * RS] = i + k;
            }
        __syncthreads();
    }
}

// B': the production tiles, but each tile stores row s's sector-aligned
// piece [t0 + d_s, t0 + TW + d_s), d_s = first 8-int boundary at or after t0
// (what a cluster exchange of <= 7 boundary slopes per row would give)
template <int TW>
__global__ void __launch_bounds__(512, 2) k_tiles_al(int* o, int nslots, int ntiles) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.y, t0 = tile * TW;
    constexpr int G = 32 / TW;
    const int sub = lane / TW, tl = lane % TW;
    for (int slot = blockIdx.z; slot < nslots; slot += gridDim.z) {
        int* base = o + slot * SLOT;
        for (int i = warp * 4 * G + sub * 4; i < H; i += 16 * 4 * G) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int s = i + k;
                const long long f = (long long)slot * SLOT + (long long)s * RS + t0;  // absolute (slot bases are not aligned)
                const int d = static_cast<int>((8 - (f & 7)) & 7);
                int t = t0 + d + tl;
                if (tile == 0 && tl < d) t = tl;  // the first tile also owns the row head
                if (s < H && t < W && (tile == 0 || t < t0 + TW + d)) base[(long long)s * RS + t] = s;
            }
        }
        __syncthreads();
    }
}

// C: full 128-byte aligned lines of the flat slot (what a perfectly
// line-shaped store would cost with the same CTA/slot walk)
__global__ void __launch_bounds__(512, 2) k_lines(int* o, int nslots, int ntiles) {
    const int tile = blockIdx.y;
    const long long per = (SLOT + ntiles - 1) / ntiles;
    for (int slot = blockIdx.z; slot < nslots; slot += gridDim.z) {
        int* base = o + slot * SLOT;
        const long long b = tile * per, e = min(SLOT, b + per);
        for (long long i = b + threadIdx.x; i < e; i += 512) base[i] = (int)i;
        __syncthreads();
    }
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int* o;
    const size_t bytes = (size_t)NSLOT * SLOT * 4;
    cudaMalloc(&o, bytes + 64);
    const double gb = bytes / 1e9;
    float t = timeit([&] { k_linear<<<148 * 8, 512>>>(reinterpret_cast<int4*>(o), bytes / 16); });
    printf("linear int4          %.4f ms  %.0f GB/s\n", t, gb / t * 1e3);
    for (int spc : {1, 4, 8}) {
        const int z = (NSLOT + spc - 1) / spc;
        t = timeit([&] { k_tiles<16><<<dim3(1, 32, z), 512>>>(o, NSLOT, 32); });
        printf("tiles16 spc=%d        %.4f ms  %.0f GB/s\n", spc, t, gb / t * 1e3);
        t = timeit([&] { k_tiles<32><<<dim3(1, 16, z), 512>>>(o, NSLOT, 16); });
        printf("tiles32 spc=%d        %.4f ms  %.0f GB/s\n", spc, t, gb / t * 1e3);
        t = timeit([&] { k_tiles_al<16><<<dim3(1, 32, z), 512>>>(o, NSLOT, 32); });
        printf("tiles16 aligned spc=%d %.4f ms  %.0f GB/s\n", spc, t, gb / t * 1e3);
        t = timeit([&] { k_tiles_al<32><<<dim3(1, 16, z), 512>>>(o, NSLOT, 16); });
        printf("tiles32 aligned spc=%d %.4f ms  %.0f GB/s\n", spc, t, gb / t * 1e3);
        t = timeit([&] { k_lines<<<dim3(1, 32, z), 512>>>(o, NSLOT, 32); });
        printf("lines   spc=%d        %.4f ms  %.0f GB/s\n", spc, t, gb / t * 1e3);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
