/*
 * fht_b200.h -- C ABI of the B200 (sm_100a) FHT2D merge-DP library
 * (paper_2411_07351_b200/libfht_b200.so).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * No exception crosses it either: every call returns an FHT_* status and
 * fht_last_error() holds the message for the calling thread.
 *
 * The reference (arXiv 2411.07351 artefact, /root/reference/proj) exposes the
 * path as C++ free functions in namespace fht; each entry point below names
 * the one it replaces.  include/fht_b200/fht.hpp rebuilds that exact C++
 * interface on top of this ABI.
 *
 * Layouts.  Images are row-major, x fastest: img[y*width + x]
 * (image.hpp:13-14, 55-58).  A quadrant's Hough image is in the reference
 * layout hough[s*W + t] (transform.cpp:80-83; W = working width = image
 * width for horiz_*, image height for vert_*), or, with FHT_LAYOUT_NATIVE,
 * slope-major hough[t*H + s].
 */
#ifndef FHT_B200_H
#define FHT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  FHT_ERR_INVALID <-> std::invalid_argument (transform.cpp:63,
 * split.hpp:34,41,54-55, image.hpp:49-53); FHT_ERR_OVERFLOW <->
 * std::overflow_error (transform.cpp:24-26). */
enum {
    FHT_OK = 0,
    FHT_ERR_INVALID = 1,
    FHT_ERR_OVERFLOW = 2,
    FHT_ERR_CUDA = 3,
    FHT_ERR_NOMEM = 4,
    FHT_ERR_INTERNAL = 5
};

/* SplitStrategy (split.hpp:12-15). */
enum { FHT_SPLIT_SIMPLE = 0, FHT_SPLIT_TWEAKED = 1 };

/* Element types. */
enum { FHT_U8 = 0, FHT_I32 = 1, FHT_I64 = 2, FHT_F32 = 3 };

/* Accumulator code for fht_plan_create: int64 accumulation whose pass 0
 * (the width-<=32 blocks) may accumulate in int32 because the caller knows
 * 32 * max|value| < 2^31 (inputs i32 / i64).  Results are identical to
 * FHT_I64; the reference-style int64 entry points choose it themselves after
 * their overflow check (transform.cpp:16-27). */
enum { FHT_I64_PASS0_I32 = FHT_I64 | 0x100 };

/* Quadrant bits, QuadrantSet order (quadrants.hpp:15-28). */
enum {
    FHT_HORIZ_POS = 1, /* fht2d(I)                       */
    FHT_HORIZ_NEG = 2, /* fht2d(flip_horizontal(I))      */
    FHT_VERT_POS = 4,  /* fht2d(transpose(I))            */
    FHT_VERT_NEG = 8,  /* fht2d(flip_horizontal(transpose(I))) */
    FHT_ALL_QUADRANTS = 15
};

/* Plan flags. */
enum {
    FHT_LAYOUT_REFERENCE = 0, /* hough[s*W + t] */
    FHT_LAYOUT_NATIVE = 1     /* hough[t*H + s] */
};

typedef struct fht_plan_s* fht_plan_t;

/* Build the integer-exact split/rounding tables for one (size, strategy)
 * once and upload them to `device`.  Valid (in, acc, out) type triples:
 *   (u8|i32, i32, i32)  (u8|i32|i64, i32, i64)  (u8|i32|i64, i64, i64)
 *   (f32|u8, f32, f32)
 * An i32 accumulator for u8 input requires W*255 < 2^31 (else
 * FHT_ERR_OVERFLOW).  `batch` images are processed per execute.  The plan's
 * tables are immutable after creation, and host threads may execute one plan
 * concurrently, each on its own stream with its own workspace and outputs
 * (the reference's transforms are safe to call concurrently):
 * the plan-owned auxiliary stream's fork/join events are recorded and waited
 * under a per-plan lock, so every call's kernels are ordered after its own
 * stream's prior work.  fht_execute_host serialises on a per-plan lock (it
 * uses plan-owned device staging buffers).
 * Replaces the per-call scratch set-up of fht::fht2d_counted
 * (transform.cpp:62-78). */
int fht_plan_create(int width, int height, int strategy, int in_dtype, int acc_dtype, int out_dtype,
                    int quadrant_mask, int batch, int layout, int device, fht_plan_t* plan);
int fht_plan_destroy(fht_plan_t plan);

/* Device workspace bytes fht_execute needs (two ping-pong buffers per
 * in-flight (image, quadrant) slot, the reference's out/tmp pair,
 * transform.cpp:75-76). */
size_t fht_workspace_bytes(fht_plan_t plan);

/* Merge additions one execute performs: count_additions_tree (oracle.cpp:27-33)
 * summed over the selected quadrants and the batch, exactly the count
 * fht2d_counted / fht2d_quadrants report (transform.cpp:56, quadrants.cpp:31). */
uint64_t fht_additions(fht_plan_t plan);

/* Kernel launches one execute issues (for the bench's gpu_launches). */
int fht_launches_per_execute(fht_plan_t plan);

/* JSON description of the schedule (blocks, halos, levels). */
int fht_plan_describe(fht_plan_t plan, char* buf, size_t len);

/* Run the transform of `batch` images on `stream` (a cudaStream_t; NULL =
 * legacy default stream).  d_in: device pointer, image i at
 * d_in + i*in_image_stride elements.  d_out[q] for quadrant bit q set in the
 * plan's mask (others ignored), image i at d_out[q] + i*out_image_stride.
 * d_workspace: fht_workspace_bytes(plan) bytes of device memory.  Stream
 * ordered, asynchronous, no host synchronisation.  No overflow check: use
 * fht_check_budget for non-u8 integer inputs.
 * Replaces fht::fht2d_quadrants (quadrants.hpp:32, quadrants.cpp:23-41) and,
 * with a single-quadrant mask, fht::fht2d (transform.hpp:36). */
int fht_execute(fht_plan_t plan, const void* d_in, int64_t in_image_stride, void* const d_out[4],
                int64_t out_image_stride, void* d_workspace, void* stream);

/* fht_execute on a pitched image view: row y of image i starts at
 * d_in + i*in_image_stride + y*in_row_pitch elements (in_row_pitch >= width).
 * Lets a plan run on a sub-image, e.g. one child subtree of the root in the
 * multi-GPU root split. */
int fht_execute_pitched(fht_plan_t plan, const void* d_in, int64_t in_row_pitch, int64_t in_image_stride,
                        void* const d_out[4], int64_t out_image_stride, void* d_workspace, void* stream);

/* fht_execute_pitched for the multi-GPU root split, with the exchange fused
 * into the transform: a one-image, one-quadrant FHT_LAYOUT_NATIVE plan whose
 * last pass also stores slopes [peer_first, peer_end) of its output to
 * d_peer + (t - peer_first) * H -- typically the other GPU's receive buffer,
 * mapped with fht_ipc_open_handle, written over NVLink as the tiles finish
 * (no separate send/recv).  d_peer = NULL: plain fht_execute_pitched. */
int fht_execute_pitched_peer(fht_plan_t plan, const void* d_in, int64_t in_row_pitch, void* const d_out[4],
                             void* d_workspace, void* d_peer, int peer_first, int peer_end, void* stream);

/* CUDA IPC for the fused exchange: export a device allocation as an opaque
 * handle (FHT_IPC_HANDLE_BYTES), open another process's handle on `device`
 * (peer access enabled on demand), close a mapping. */
#define FHT_IPC_HANDLE_BYTES 64
/* A dedicated cudaMalloc allocation (an IPC handle covers a whole allocation,
 * so exported buffers must not be sub-allocated). */
int fht_device_alloc(size_t bytes, int device, void** d_ptr);
int fht_device_free(void* d_ptr);
int fht_ipc_get_handle(const void* d_ptr, void* handle, size_t handle_len);
int fht_ipc_open_handle(const void* handle, size_t handle_len, int device, void** d_ptr);
int fht_ipc_close(void* d_ptr);

/* The root level of a width-W, H-shift transform from its two children, each
 * given as a slope-major column range (the FHT_LAYOUT_NATIVE output of a plan
 * over that child's columns): left child slopes [left_first, ...) at d_left,
 * right child slopes [right_first, ...) at d_right, column stride H.  Writes
 * root slopes [t_begin, t_end) of d_out (reference layout hough[s*W + t] or
 * native hough[t*H + s]):  OUT[t][s] = L[t0][s] + R[t1][(s + r) mod H]
 * (transform.cpp:46-57).  Used by the multi-GPU root split, where each GPU
 * owns one child and merges half the root.  Stream ordered and asynchronous:
 * the slope table is built once per (width, height, strategy, device) and
 * cached on the device. */
int fht_merge_root(int width, int height, int strategy, int acc_dtype, int out_dtype, int layout, const void* d_left,
                   int left_first, const void* d_right, int right_first, int t_begin, int t_end, void* d_out,
                   void* stream);

/* fht_execute with a CUDA event recorded after every kernel launch on
 * `stream`; synchronises and returns each launch's duration (ms), kind
 * (5 = u8 staging, 1 = K1 generic blocks, 4 = K1P width-32 Brady-Yong blocks,
 * 2 = K2 fused upper pass, 3 = K2 root pass) and algorithmic bytes (each input cell read
 * once, each output cell written once).  For the bench's live per-kernel
 * roofline. */
int fht_execute_profiled(fht_plan_t plan, const void* d_in, int64_t in_image_stride, void* const d_out[4],
                         int64_t out_image_stride, void* d_workspace, void* stream, float* launch_ms,
                         int* launch_kind, double* launch_bytes, int max_launches, int* n_launches);

/* Same, with HOST buffers: copies the inputs host->device, runs, copies the
 * outputs device->host and synchronises `stream`.  Uses device staging
 * buffers owned by the plan (serialised by a per-plan mutex).  Images and
 * outputs are dense (strides = one image). */
int fht_execute_host(fht_plan_t plan, const void* h_in, void* const h_out[4], void* stream);

/* check_overflow_budget (transform.cpp:16-27) on device data: *ok_for_i32 =
 * (width * max|v| < 2^31), returns FHT_ERR_OVERFLOW if width * max|v| >= 2^62.
 * Synchronises `stream`. */
int fht_check_budget(const void* d_in, int dtype, int64_t count, int width, int* ok_for_i32, void* stream);

/* The reference entry points with host int64 buffers, bit-exact:
 *   fht_fht2d_counted_i64  <-> fht::fht2d_counted (transform.hpp:40)
 *   fht_fht2d_quadrants_i64 <-> fht::fht2d_quadrants (quadrants.hpp:32-33)
 * The overflow budget is checked on the device (FHT_ERR_OVERFLOW as the
 * reference's overflow_error); accumulation is int32 when
 * width * max|v| < 2^31 and int64 otherwise.  Plans are cached per device. */
int fht_fht2d_counted_i64(const int64_t* img, int width, int height, int strategy, int64_t* hough,
                          uint64_t* additions);
int fht_fht2d_quadrants_i64(const int64_t* img, int width, int height, int strategy, int64_t* horiz_pos,
                            int64_t* horiz_neg, int64_t* vert_pos, int64_t* vert_neg,
                            uint64_t* total_additions);

/* Structure-free validation path (the reference's oracle, oracle.cpp:9-25):
 * J(t, s) = sum_x I(x, (pat_t(x) + s) mod h) by direct Theta(w^2 h)
 * summation on the device with Algorithm-2 patterns (pattern.cpp:10-30),
 * int64 accumulation, reference layout.  For checking the fast path at sizes
 * where a CPU oracle is infeasible.
 *   fht_slow_hough_device: integer image on the device (dtype FHT_U8 / FHT_I32
 *     / FHT_I64), quadrant code 0..3 (QuadrantSet order), int64 output on the
 *     device; stream ordered.
 *   fht_slow_hough_i64 <-> fht::slow_hough (oracle.hpp:17), host buffers. */
int fht_slow_hough_device(const void* d_img, int in_dtype, int width, int height, int strategy, int quadrant,
                          int64_t* d_hough, void* stream);
int fht_slow_hough_i64(const int64_t* img, int width, int height, int strategy, int64_t* hough);

/* Algorithm 2: the slope-t generating pattern of width n (n values)
 * <-> fht::fht2d_pattern (pattern.hpp:20, pattern.cpp:24-30). */
int fht_fht2d_pattern(int n, int t, int strategy, int* values);

/* The paper's accuracy sweep on the device (analysis.cpp:63-91): for each
 * width n in [n_lo, n_hi] (<= 46340), worst[n - n_lo] = max over slopes t and
 * columns x of |x t - pat(n,t)(x) (n-1)|, i.e. E(n) = worst / (n-1) exactly
 * (max_orthotropic_error, analysis.hpp:39).  Synchronous. */
int fht_max_deviation_numerators(int n_lo, int n_hi, int strategy, int64_t* worst);

/* Host helpers, identical to the reference's integer rules. */
int fht_split_width(int w, int strategy, int* w0, int* w1);                 /* split.hpp:46-48 */
int fht_round_half_up_ratio(int64_t num, int64_t den, int64_t* result);     /* split.hpp:53-57 */
int fht_count_additions_tree(int w, int h, int strategy, uint64_t* result); /* oracle.cpp:27-33 */

/* Host-only export of the schedule tables for one working orientation
 * (W slopes x H shifts) as JSON: blocks [x0, shape, depth], shapes {width,
 * steps, halo, step_offset, ops [dst, a, b, shift, extra]} and the fused
 * upper passes {levels, tiles, loads, step_offs, ops, stores}.  Needs no GPU;
 * used by the CPU tests that replay the schedule against the oracle.
 * Returns FHT_ERR_INVALID if `len` is too small (then *needed holds the size). */
int fht_schedule_json(int W, int H, int strategy, int block_width, int pass_levels, int tile_width, char* buf,
                      size_t len, size_t* needed);

/* The plans behind fht_fht2d_counted_i64 / fht_fht2d_quadrants_i64 are cached
 * per (size, strategy, accumulator, quadrants, device), least recently used
 * first out, at most FHT_PLAN_CACHE (environment, default 8).  Release them
 * all (e.g. before cudaDeviceReset); *released (may be NULL) = how many.
 * Plans a concurrent call is still using are freed when it returns. */
int fht_plan_cache_clear(size_t* released);
size_t fht_plan_cache_size(void);

/* Diagnostics: the stream synchronisations and device allocations this
 * library has made so far (process-wide).  Lets a test check that a timed
 * step -- an execute, or the multi-GPU root split's child + merge -- makes
 * neither. */
int fht_debug_counters(uint64_t* host_syncs, uint64_t* device_allocs);

/* Message of the last failed call on this thread ("" if none). */
const char* fht_last_error(void);

/* Library version string. */
const char* fht_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FHT_B200_H */
