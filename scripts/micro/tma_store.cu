// Micro-test: 2D TMA tensor store of a [rows][16] int32 box from shared
// memory into a 4-row lattice view of a row-major [N][W] int32 array
// (W = 509: row stride 2036 B is not a multiple of 16, the lattice stride
// 4 * 2036 is).  Checks (a) smem sources aligned to 16 (not 128) bytes,
// (b) correctness, (c) time of many small stores.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_store(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm1, int W, int nrows_img, int nimg, int align_off, int flags) {
    extern __shared__ __align__(1024) unsigned char smem[];
    // one CTA per (image, 16-slope tile); smem: 4 regions (row residues) of 128 rows x 64 B
    const int tile = blockIdx.x, img = blockIdx.y;
    const int t0 = tile * 16;
    int* st = reinterpret_cast<int*>(smem + align_off);
    const int R = (nrows_img + 3) / 4;
    for (int i = threadIdx.x; i < 4 * R * 16; i += blockDim.x) {
        const int rho = i / (R * 16), j = (i / 16) % R, tl = i % 16;
        const int s = 4 * j + rho;
        st[i] = (s < nrows_img && t0 + tl < W) ? (img * 1000000 + s * 1000 + t0 + tl) : -1;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0 && !(flags & 4)) {
        for (int rho = 0; rho < ((flags & 8) ? 1 : 4); ++rho) {
            const long long Rg = (long long)img * nrows_img + rho;  // global row of j = 0
            const int n = (nrows_img - rho + 3) / 4;
            const int y0 = (int)(Rg >> 2), x0 = (int)((Rg & 3) * W + t0);
            for (int j = 0; j < ((flags & 8) ? 1 : n); j += 64) {
                const int jj = (j + 64 <= n) ? j : ((n - 64) & ~1);
                const unsigned src = (unsigned)__cvta_generic_to_shared(st + (rho * R + jj) * 16);
                if (flags & 2)
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
                                 :: "l"(reinterpret_cast<unsigned long long>(&tm)), "r"(x0), "r"(y0 + jj), "r"(src) : "memory");
                else
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                 :: "l"(&tm), "r"(x0), "r"(y0 + jj), "r"(src) : "memory");
                if (jj + 64 == n - 1 && !(flags & 1)) {  // the one row an even-aligned 64-row box leaves
                    const unsigned s1 = (unsigned)__cvta_generic_to_shared(st + (rho * R + n - 1) * 16);
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                 :: "l"(&tm1), "r"(x0), "r"(y0 + n - 1), "r"(s1) : "memory");
                }
            }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncthreads();
}

int main(int argc, char** argv) {
    const int W = 509, H = 509, nimg = argc > 1 ? atoi(argv[1]) : 64, align_off = argc > 2 ? atoi(argv[2]) : 16, flags = argc > 3 ? atoi(argv[3]) : 0;
    const long long N = (long long)nimg * H * W;
    int* d;
    CK(cudaMalloc(&d, N * 4));
    CK(cudaMemset(d, 0xff, N * 4));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)4 * W, (cuuint64_t)(nimg * H / 4)};
    cuuint64_t strides[1] = {(cuuint64_t)16 * W};
    cuuint32_t box[2] = {16, 64};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    CUtensorMap tm1;
    cuuint32_t box1[2] = {16, 1};
    r = enc(&tm1, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, d, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode1: %d\n", (int)r);
    const int smem = 4 * 128 * 64 + 1024;
    CK(cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 g((W + 15) / 16, nimg);
    k_store<<<g, 256, smem>>>(tm, tm1, W, H, nimg, align_off, flags);
    CK(cudaDeviceSynchronize());
    std::vector<int> h(N);
    CK(cudaMemcpy(h.data(), d, N * 4, cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (int i = 0; i < nimg; ++i)
        for (int s = 0; s < H; ++s)
            for (int t = 0; t < W; ++t) {
                const int v = h[((long long)i * H + s) * W + t];
                if (v != i * 1000000 + s * 1000 + t) { if (bad < 5) printf("bad i%d s%d t%d: %d\n", i, s, t, v); ++bad; }
            }
    printf("align_off %d: bad %lld of %lld\n", align_off, bad, N);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) k_store<<<g, 256, smem>>>(tm, tm1, W, H, nimg, align_off, flags);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("time per launch %.4f ms (%.1f GB/s of output, %d CTAs, %d TMA ops each)\n", ms / 10, N * 4 / (ms / 10 * 1e-3) / 1e9, g.x * g.y, 4 * 2);
    return 0;
}
