// slow.cuh -- device slow_hough (oracle.cpp:9-25), see slow.cu.
#pragma once

#include <cuda_runtime.h>

namespace fhtb {
// Quadrant q of an integer image (in_dtype 0 u8, 1 i32, 2 i64) -> int64
// Hough image in the reference layout.  d_pat: W x W patterns (row t);
// d_cols: W*H int64 scratch.
void launch_slow_hough(const void* img, int in_dtype, int img_w, int img_h, int q, const int* d_pat, int W, int H,
                       long long* d_cols, long long* d_out, cudaStream_t st);
// Max orthotropic error numerators for n in [n_lo, n_hi] (analysis.cpp:63-91)
// into d_worst[n - n_lo] (must be zeroed).
void launch_max_deviation(int n_lo, int n_hi, int strategy, unsigned long long* d_worst, cudaStream_t st);
}  // namespace fhtb
