// Minimal TMA tensor load + store round trip (diagnostic).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k(const __grid_constant__ CUtensorMap tm, int mode) {
    __shared__ __align__(128) int buf[64 * 16];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(buf), bb = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (mode & 1) {  // load
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bb), "r"(64 * 16 * 4));
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         :: "r"(sb), "l"(&tm), "r"(0), "r"(0), "r"(bb) : "memory");
        }
        unsigned done = 0;
        while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bb));
    } else {
        for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) buf[i] = i;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) buf[i] += 1;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if ((mode & 2) && threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" :: "l"(&tm), "r"(16), "r"(0), "r"(sb) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main(int argc, char** argv) {
    const int mode = atoi(argv[1]), W = atoi(argv[2]), rows = 256;
    int* d; CK(cudaMalloc(&d, (size_t)W * rows * 4)); CK(cudaMemset(d, 0, (size_t)W * rows * 4));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)W * 4};
    cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("mode %d W %d encode %d q %d\n", mode, W, (int)r, (int)q);
    k<<<1, 128>>>(tm, mode);
    CK(cudaDeviceSynchronize());
    int h[4]; CK(cudaMemcpy(h, d + 16, 16, cudaMemcpyDeviceToHost));
    printf("ok %d %d %d %d\n", h[0], h[1], h[2], h[3]);
}
