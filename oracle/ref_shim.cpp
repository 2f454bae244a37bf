// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference sources where they lie under
// /root/reference/proj/src (transform.cpp, quadrants.cpp, pattern.cpp,
// oracle.cpp) into oracle/_ref/libfhtref.so.  Nothing is copied: the shim
// only converts plain pointers into fht::Image values and calls the
// reference's own public API:
//   fht::fht2d_counted     transform.hpp:40   (transform.cpp:62-85)
//   fht::fht2d_quadrants   quadrants.hpp:32   (quadrants.cpp:23-41)
//   fht::slow_hough        oracle.hpp:17      (oracle.cpp:9-25)
//   fht::fht2d_pattern     pattern.hpp:20     (pattern.cpp:24-30)
//   fht::count_additions_tree oracle.hpp:22   (oracle.cpp:27-33)
// Exceptions are mapped to status codes: 1 invalid_argument, 2
// overflow_error, 4 anything else; the message goes to `err`.
//
// ref_batch_quadrants_u8 is the CPU baseline used by bench.py: it runs the
// reference's per-quadrant transforms on a batch of uint8 images with a pool
// of host threads over (image, quadrant) items (the reference is safe to call
// concurrently).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fht/analysis.hpp"
#include "fht/oracle.hpp"
#include "fht/pattern.hpp"
#include "fht/quadrants.hpp"
#include "fht/transform.hpp"

namespace {

void set_err(char* err, int errlen, const char* what) {
    if (!err || errlen <= 0) return;
    std::strncpy(err, what, static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = '\0';
}

template <class F>
int guarded(char* err, int errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const std::overflow_error& e) {
        set_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 4;
    }
}

fht::SplitStrategy strat(int s) { return s == 0 ? fht::SplitStrategy::Simple : fht::SplitStrategy::Tweaked; }

void copy_out(const fht::HoughImage& h, int64_t* out) {
    std::memcpy(out, h.data().data(), h.data().size() * sizeof(int64_t));
}

}  // namespace

extern "C" {

int ref_fht2d_counted(const int64_t* img, int w, int h, int strategy, int64_t* hough,
                      uint64_t* additions, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        std::vector<int64_t> v;
        if (w > 0 && h > 0) v.assign(img, img + static_cast<std::size_t>(w) * h);
        fht::Image im = (w > 0 && h > 0) ? fht::Image(w, h, std::move(v)) : fht::Image();
        fht::CountedTransform r = fht::fht2d_counted(im, strat(strategy));
        copy_out(r.hough, hough);
        if (additions) *additions = r.additions;
    });
}

int ref_fht2d_quadrants(const int64_t* img, int w, int h, int strategy, int64_t* horiz_pos,
                        int64_t* horiz_neg, int64_t* vert_pos, int64_t* vert_neg,
                        uint64_t* total_additions, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        fht::Image im(w, h, std::vector<int64_t>(img, img + static_cast<std::size_t>(w) * h));
        fht::QuadrantSet q = fht::fht2d_quadrants(im, strat(strategy), total_additions);
        copy_out(q.horiz_pos, horiz_pos);
        copy_out(q.horiz_neg, horiz_neg);
        copy_out(q.vert_pos, vert_pos);
        copy_out(q.vert_neg, vert_neg);
    });
}

int ref_slow_hough(const int64_t* img, int w, int h, int strategy, int64_t* hough, char* err,
                   int errlen) {
    return guarded(err, errlen, [&] {
        fht::Image im(w, h, std::vector<int64_t>(img, img + static_cast<std::size_t>(w) * h));
        copy_out(fht::slow_hough(im, strat(strategy)), hough);
    });
}

int ref_fht2d_pattern(int n, int t, int strategy, int* values, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        fht::Pattern p = fht::fht2d_pattern(n, t, strat(strategy));
        std::memcpy(values, p.values.data(), p.values.size() * sizeof(int));
    });
}

uint64_t ref_count_additions_tree(int w, int h, int strategy) {
    return fht::count_additions_tree(w, h, strat(strategy));
}

// CPU baseline: n_img uint8 images (image i at img + i*w*h), the quadrants
// in quadrant_mask, widened to int64 and transformed by the reference:
// work items (image, quadrant) are pulled from a shared counter by `threads`
// host threads (concurrent calls are safe), so a single
// image's four quadrants also run in parallel.  Item (i, q) runs
// fht2d_counted on the same flipped / transposed input fht2d_quadrants
// builds (quadrants.cpp:25-37).  If `out` is non-null image i's quadrant q
// goes to out + (i*4 + q)*w*h.
int ref_batch_quadrants_u8(const uint8_t* img, int n_img, int w, int h, int strategy,
                           int quadrant_mask, int threads, int64_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const std::size_t cells = static_cast<std::size_t>(w) * h;
        std::vector<int> quads;
        for (int q = 0; q < 4; ++q)
            if (quadrant_mask & (1 << q)) quads.push_back(q);
        // whole images per work item once there are enough of them: then
        // each item is exactly the reference's own fht2d_quadrants (one
        // transpose per image, quadrants.cpp:23-41); fewer images than
        // threads: (image, quadrant) items, so one image's quadrants run in
        // parallel
        const bool per_image = quadrant_mask == 15 && n_img >= std::max(1, threads);
        const int n_items = per_image ? n_img : n_img * static_cast<int>(quads.size());
        std::atomic<int> next{0};
        std::atomic<int> failed{0};
        std::string first_error;
        auto worker = [&] {
            for (;;) {
                const int k = next.fetch_add(1);
                if (k >= n_items || failed.load()) return;
                try {
                    if (per_image) {
                        std::vector<int64_t> v(cells);
                        const uint8_t* src = img + static_cast<std::size_t>(k) * cells;
                        for (std::size_t c = 0; c < cells; ++c) v[c] = src[c];
                        fht::QuadrantSet qs = fht::fht2d_quadrants(fht::Image(w, h, std::move(v)), strat(strategy));
                        if (out) {
                            int64_t* o = out + static_cast<std::size_t>(k) * 4 * cells;
                            copy_out(qs.horiz_pos, o);
                            copy_out(qs.horiz_neg, o + cells);
                            copy_out(qs.vert_pos, o + 2 * cells);
                            copy_out(qs.vert_neg, o + 3 * cells);
                        }
                        continue;
                    }
                    const int i = k / static_cast<int>(quads.size()), q = quads[static_cast<std::size_t>(k) % quads.size()];
                    std::vector<int64_t> v(cells);
                    const uint8_t* src = img + static_cast<std::size_t>(i) * cells;
                    for (std::size_t c = 0; c < cells; ++c) v[c] = src[c];
                    fht::Image im(w, h, std::move(v));
                    fht::Image input;
                    if (q == 0) input = std::move(im);
                    else if (q == 1) input = fht::flip_horizontal(im);
                    else if (q == 2) input = fht::transpose(im);
                    else input = fht::flip_horizontal(fht::transpose(im));
                    fht::CountedTransform r = fht::fht2d_counted(input, strat(strategy));
                    if (out) copy_out(r.hough, out + (static_cast<std::size_t>(i) * 4 + q) * cells);
                } catch (const std::exception& e) {
                    if (!failed.exchange(1)) first_error = e.what();
                    return;
                }
            }
        };
        const int nt = std::max(1, std::min(threads, n_items));
        std::vector<std::thread> pool;
        for (int k = 1; k < nt; ++k) pool.emplace_back(worker);
        worker();
        for (auto& t : pool) t.join();
        if (failed.load()) throw std::runtime_error(first_error);
    });
}

// transform.cpp:8-14: u(i) = v((i + r) mod h)
int ref_rotate(const int64_t* v, int h, int r, int64_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const std::vector<fht::Accum> u = fht::rotate(std::span<const fht::Accum>(v, static_cast<std::size_t>(h)), r);
        std::memcpy(out, u.data(), u.size() * sizeof(int64_t));
    });
}

// analysis.hpp:37-62 (paper-figure reproduction): exact rationals as (num, den).
int ref_max_orthotropic_error(int n, int strategy, int64_t* num, int64_t* den, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const fht::Rational r = fht::max_orthotropic_error(n, strat(strategy));
        *num = r.num();
        *den = r.den();
    });
}

int ref_separation_fraction(int n_max, int threads, int64_t* num, int64_t* den, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const fht::Rational r = fht::separation_fraction(n_max, static_cast<unsigned>(threads));
        *num = r.num();
        *den = r.den();
    });
}

int ref_tweaked_error_bound(int n, int64_t* num, int64_t* den, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const fht::Rational r = fht::tweaked_error_bound(n);
        *num = r.num();
        *den = r.den();
    });
}

}  // extern "C"
