/*
 * fht_oracle.c -- CPU restatement of the reference FHT2D merge DP.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2411_07351_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never calls into it (it fails loudly if its CUDA library is missing).
 *
 * It restates, function by function, the reference at /root/reference/proj:
 *   split_simple / split_tweaked / split_width   include/fht/split.hpp:33-48
 *   round_half_up_ratio                          include/fht/split.hpp:53-57
 *   transform_columns (recursive merge DP)       src/transform.cpp:35-58
 *   fht2d_counted (layout conversion + driver)   src/transform.cpp:62-85
 *   check_overflow_budget                        src/transform.cpp:16-27
 *   flip_horizontal / transpose / fht2d_quadrants src/quadrants.cpp:7-41
 *   fht2d_pattern (Algorithm 2)                  src/pattern.cpp:10-30
 *   slow_hough                                   src/oracle.cpp:9-25
 *   count_additions_tree                         src/oracle.cpp:27-33
 *
 * The reference only has an int64 path (image.hpp:11).  The float32 and
 * float64 instantiations follow the identical add tree (same split, same
 * rounding, same A+B operand pairing and wrap), which is what the BASELINE
 * float configs are checked against.  Build with -ffp-contract=off and no
 * fast-math so the fp32 adds are exactly the IEEE adds of the tree.
 *
 * Parity pinning: the int64 instantiation is checked bit-exactly against the
 * reference library compiled from /root/reference (oracle/_ref) and against
 * the golden fixtures under tests/golden/ that the reference generated
 * (tests/golden/make_golden.py); see tests/test_oracle.py.
 *
 * Return codes: 0 ok, 1 invalid argument (std::invalid_argument in the
 * reference), 2 overflow (std::overflow_error), 3 out of memory.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FHT_OK 0
#define FHT_EINVAL 1
#define FHT_EOVERFLOW 2
#define FHT_ENOMEM 3

/* split.hpp:33-48 */
static int oracle_split(int w, int strategy, int* w0, int* w1) {
    if (w < 2) return FHT_EINVAL;
    if (strategy == 0) { /* Simple: (floor(w/2), ceil(w/2)) */
        *w0 = w / 2;
    } else { /* Tweaked: largest power of two strictly below w */
        unsigned v = (unsigned)(w - 1);
        int bw = 0;
        while (v) { ++bw; v >>= 1; }
        *w0 = 1 << (bw - 1);
    }
    *w1 = w - *w0;
    return FHT_OK;
}

int oracle_split_width(int w, int strategy, int* w0, int* w1) { return oracle_split(w, strategy, w0, w1); }

/* split.hpp:53-57: floor((2 num + den) / (2 den)), ties rounded up. */
static int64_t oracle_rhu(int64_t num, int64_t den) { return (2 * num + den) / (2 * den); }

int64_t oracle_round_half_up_ratio(int64_t num, int64_t den) { return oracle_rhu(num, den); }

/* transform.cpp:16-27 (only meaningful for the int64 instantiation). */
int oracle_check_overflow_budget(const int64_t* data, int w, int h) {
    uint64_t vmax = 0;
    size_t n = (size_t)w * (size_t)h;
    for (size_t i = 0; i < n; ++i) {
        int64_t v = data[i];
        uint64_t a = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
        if (a > vmax) vmax = a;
    }
    unsigned __int128 budget = (unsigned __int128)1 << 62;
    if ((unsigned __int128)(unsigned)w * vmax >= budget) return FHT_EOVERFLOW;
    return FHT_OK;
}

/*
 * transform.cpp:35-58, restated per element type.  `in` is the column-major
 * scratch (column x at [x*h, (x+1)*h)); `out` receives the transform, `tmp`
 * is scratch and the roles swap one level down (43-44).
 */
#define DEFINE_ORACLE_TRANSFORM(T, SUF)                                                         \
    static void cols_##SUF(const T* in, T* out, T* tmp, int w, int h, int strategy,             \
                           uint64_t* additions) {                                               \
        if (w == 1) { /* leaf: copy (37-40) */                                                  \
            memcpy(out, in, sizeof(T) * (size_t)h);                                             \
            return;                                                                             \
        }                                                                                       \
        int w0 = 0, w1 = 0;                                                                     \
        oracle_split(w, strategy, &w0, &w1);                                                    \
        size_t left = (size_t)w0 * (size_t)h;                                                   \
        cols_##SUF(in, tmp, out, w0, h, strategy, additions);                                   \
        cols_##SUF(in + left, tmp + left, out + left, w1, h, strategy, additions);              \
        for (int t = 0; t < w; ++t) { /* merge (46-57) */                                       \
            int64_t t0 = oracle_rhu((int64_t)t * (w0 - 1), w - 1);                             \
            int64_t t1 = oracle_rhu((int64_t)t * (w1 - 1), w - 1);                              \
            int r = (int)((t - t1) % h);                                                        \
            const T* a = tmp + (size_t)t0 * h;                                                  \
            const T* b = tmp + ((size_t)w0 + (size_t)t1) * h;                                   \
            T* dst = out + (size_t)t * h;                                                       \
            int wrap = h - r;                                                                   \
            for (int s = 0; s < wrap; ++s) dst[s] = a[s] + b[s + r];                            \
            for (int s = wrap; s < h; ++s) dst[s] = a[s] + b[s + r - h];                        \
            *additions += (uint64_t)h;                                                          \
        }                                                                                       \
    }                                                                                           \
    /* transform.cpp:62-85: row-major image in, row-major Hough image [s][t] out. */            \
    int oracle_fht2d_##SUF(const T* img, int w, int h, int strategy, T* hough,                 \
                           uint64_t* additions) {                                               \
        if (w < 1 || h < 1) return FHT_EINVAL;                                                  \
        if (strategy != 0 && strategy != 1) return FHT_EINVAL;                                  \
        size_t cells = (size_t)w * (size_t)h;                                                   \
        T* cols = (T*)malloc(sizeof(T) * cells);                                                \
        T* out = (T*)malloc(sizeof(T) * cells);                                                 \
        T* tmp = (T*)malloc(sizeof(T) * cells);                                                 \
        if (!cols || !out || !tmp) {                                                            \
            free(cols); free(out); free(tmp);                                                   \
            return FHT_ENOMEM;                                                                  \
        }                                                                                       \
        for (int y = 0; y < h; ++y)                                                             \
            for (int x = 0; x < w; ++x) cols[(size_t)x * h + y] = img[(size_t)y * w + x];       \
        uint64_t adds = 0;                                                                      \
        cols_##SUF(cols, out, tmp, w, h, strategy, &adds);                                      \
        for (int t = 0; t < w; ++t)                                                             \
            for (int s = 0; s < h; ++s) hough[(size_t)s * w + t] = out[(size_t)t * h + s];      \
        if (additions) *additions = adds;                                                       \
        free(cols); free(out); free(tmp);                                                       \
        return FHT_OK;                                                                          \
    }                                                                                           \
    /* quadrants.cpp:23-41 with flip_horizontal (7-13) and transpose (15-21) as copies. */      \
    int oracle_fht2d_quadrants_##SUF(const T* img, int w, int h, int strategy, T* horiz_pos,    \
                                     T* horiz_neg, T* vert_pos, T* vert_neg,                    \
                                     uint64_t* total_additions) {                               \
        if (w < 1 || h < 1) return FHT_EINVAL;                                                  \
        size_t cells = (size_t)w * (size_t)h;                                                   \
        T* tr = (T*)malloc(sizeof(T) * cells);                                                  \
        T* fl = (T*)malloc(sizeof(T) * cells);                                                  \
        if (!tr || !fl) { free(tr); free(fl); return FHT_ENOMEM; }                              \
        for (int y = 0; y < h; ++y) /* transpose: out(y,x) = img(x,y); out is h wide */         \
            for (int x = 0; x < w; ++x) tr[(size_t)x * h + y] = img[(size_t)y * w + x];        \
        uint64_t total = 0, adds = 0;                                                           \
        int rc = oracle_fht2d_##SUF(img, w, h, strategy, horiz_pos, &adds);                     \
        total += adds;                                                                          \
        for (int y = 0; rc == 0 && y < h; ++y)                                                  \
            for (int x = 0; x < w; ++x) fl[(size_t)y * w + x] = img[(size_t)y * w + (w - 1 - x)]; \
        if (rc == 0) rc = oracle_fht2d_##SUF(fl, w, h, strategy, horiz_neg, &adds);             \
        total += adds;                                                                          \
        if (rc == 0) rc = oracle_fht2d_##SUF(tr, h, w, strategy, vert_pos, &adds);              \
        total += adds;                                                                          \
        for (int y = 0; rc == 0 && y < w; ++y) /* flip of the transposed image (h wide) */      \
            for (int x = 0; x < h; ++x) fl[(size_t)y * h + x] = tr[(size_t)y * h + (h - 1 - x)]; \
        if (rc == 0) rc = oracle_fht2d_##SUF(fl, h, w, strategy, vert_neg, &adds);              \
        total += adds;                                                                          \
        if (total_additions) *total_additions = total;                                          \
        free(tr); free(fl);                                                                     \
        return rc;                                                                              \
    }

DEFINE_ORACLE_TRANSFORM(int64_t, i64)
DEFINE_ORACLE_TRANSFORM(int32_t, i32)
DEFINE_ORACLE_TRANSFORM(float, f32)
DEFINE_ORACLE_TRANSFORM(double, f64)

/* The reference entry point proper: int64 with the overflow budget (transform.cpp:62-64). */
int oracle_fht2d_counted(const int64_t* img, int w, int h, int strategy, int64_t* hough,
                         uint64_t* additions) {
    if (w < 1 || h < 1) return FHT_EINVAL;
    int rc = oracle_check_overflow_budget(img, w, h);
    if (rc) return rc;
    return oracle_fht2d_i64(img, w, h, strategy, hough, additions);
}

/* pattern.cpp:10-20 (build_values) and 24-30 (fht2d_pattern). */
static void build_values(int* out, int n, int t, int lift, int strategy) {
    if (n == 1) {
        out[0] = lift;
        return;
    }
    int n0 = 0, n1 = 0;
    oracle_split(n, strategy, &n0, &n1);
    int t0 = (int)oracle_rhu((int64_t)t * (n0 - 1), n - 1);
    int t1 = (int)oracle_rhu((int64_t)t * (n1 - 1), n - 1);
    build_values(out, n0, t0, lift, strategy);
    build_values(out + n0, n1, t1, lift + (t - t1), strategy);
}

int oracle_fht2d_pattern(int n, int t, int strategy, int* values) {
    if (n < 1 || t < 0 || t >= n) return FHT_EINVAL;
    build_values(values, n, t, 0, strategy);
    return FHT_OK;
}

/* oracle.cpp:9-25: direct Theta(w^2 h) summation along every shifted pattern. */
int oracle_slow_hough_i64(const int64_t* img, int w, int h, int strategy, int64_t* hough) {
    if (w < 1 || h < 1) return FHT_EINVAL;
    int rc = oracle_check_overflow_budget(img, w, h);
    if (rc) return rc;
    int* pat = (int*)malloc(sizeof(int) * (size_t)w);
    if (!pat) return FHT_ENOMEM;
    for (int t = 0; t < w; ++t) {
        build_values(pat, w, t, 0, strategy);
        for (int s = 0; s < h; ++s) {
            int64_t sum = 0;
            for (int x = 0; x < w; ++x) sum += img[(size_t)((pat[x] + s) % h) * w + x];
            hough[(size_t)s * w + t] = sum;
        }
    }
    free(pat);
    return FHT_OK;
}

/* oracle.cpp:27-33 */
uint64_t oracle_count_additions_tree(int w, int h, int strategy) {
    if (w < 1 || h < 1) return 0;
    if (w == 1) return 0;
    int w0, w1;
    oracle_split(w, strategy, &w0, &w1);
    return (uint64_t)w * (uint64_t)h + oracle_count_additions_tree(w0, h, strategy) +
           oracle_count_additions_tree(w1, h, strategy);
}

/*
 * CPU-baseline helper (port flavour of oracle/ref_shim.cpp's
 * ref_batch_quadrants_u8): n_img uint8 images, the quadrants in
 * quadrant_mask, widened to int64, `threads` pthreads over (image, quadrant)
 * items.  If out is non-null image i's quadrant q goes to out + (i*4+q)*w*h.
 */
#include <pthread.h>

typedef struct {
    const uint8_t* img;
    int n_img, w, h, strategy, mask;
    int64_t* out;
    int next;
    int rc;
    pthread_mutex_t mu;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    size_t cells = (size_t)j->w * (size_t)j->h;
    int quads[4], nq = 0;
    for (int q = 0; q < 4; ++q)
        if (j->mask & (1 << q)) quads[nq++] = q;
    int64_t* in = (int64_t*)malloc(sizeof(int64_t) * cells);
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * cells);
    int64_t* res = (int64_t*)malloc(sizeof(int64_t) * cells);
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int k = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (k >= j->n_img * nq) break;
        int i = k / nq, q = quads[k % nq];
        const uint8_t* src = j->img + (size_t)i * cells;
        int W = j->w, H = j->h;
        /* the quadrant's input as fht2d_quadrants builds it (quadrants.cpp:25-37) */
        for (int y = 0; y < j->h; ++y)
            for (int x = 0; x < j->w; ++x) {
                int64_t v = src[(size_t)y * j->w + x];
                if (q == 0) in[(size_t)y * j->w + x] = v;
                else if (q == 1) in[(size_t)y * j->w + (j->w - 1 - x)] = v;
                else if (q == 2) in[(size_t)x * j->h + y] = v;
                else in[(size_t)x * j->h + (j->h - 1 - y)] = v;
            }
        if (q >= 2) { W = j->h; H = j->w; }
        (void)tmp;
        int rc = oracle_fht2d_i64(in, W, H, j->strategy, res, 0);
        if (rc) { j->rc = rc; break; }
        if (j->out) memcpy(j->out + ((size_t)i * 4 + q) * cells, res, sizeof(int64_t) * cells);
    }
    free(in);
    free(tmp);
    free(res);
    return 0;
}

int oracle_batch_quadrants_u8(const uint8_t* img, int n_img, int w, int h, int strategy,
                              int quadrant_mask, int threads, int64_t* out) {
    batch_job j = {img, n_img, w, h, strategy, quadrant_mask, out, 0, 0, PTHREAD_MUTEX_INITIALIZER};
    int nt = threads < 1 ? 1 : threads;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
    for (int k = 1; k < nt; ++k) pthread_create(&tid[k], 0, batch_worker, &j);
    batch_worker(&j);
    for (int k = 1; k < nt; ++k) pthread_join(tid[k], 0);
    free(tid);
    return j.rc;
}
