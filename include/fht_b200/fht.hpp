// fht_b200/fht.hpp -- the reference's C++ interface for the FHT2D path,
// rebuilt header-only on the C ABI (include/fht_b200.h), so that code written
// against the reference library (namespace fht, /root/reference/proj/include/fht)
// can switch to the B200 implementation by changing its include and link line:
//
//     #include "fht_b200/fht.hpp"
//     namespace fht = fht_b200;          // or: #include "fht_b200/as_fht.hpp"
//     ... link -lfht_b200 (paper_2411_07351_b200/libfht_b200.so)
//
// Same types, names, argument meaning, layouts and exception types:
//   Accum, Image, HoughImage             image.hpp:11-68
//   SplitStrategy, to_string, strategy_from_string, floor_log2,
//   split_simple, split_tweaked, split_width, round_half_up_ratio
//                                        split.hpp:12-57
//   rotate, check_overflow_budget, CountedTransform, fht2d, fht2d_counted
//                                        transform.hpp:12-40
//   flip_horizontal, transpose, QuadrantSet, fht2d_quadrants
//                                        quadrants.hpp:10-33
//   Pattern, fht2d_pattern, pattern_set  pattern.hpp:12-24
//   slow_hough, count_additions_tree     oracle.hpp:15-22
// fht2d / fht2d_counted / fht2d_quadrants run on the current CUDA device;
// the overflow budget is checked there (std::overflow_error as in
// transform.cpp:24-26).  Plan is the batched, device-resident interface.
#pragma once

#include <bit>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../fht_b200.h"

namespace fht_b200 {

// ----------------------------------------------------------------- errors
inline void throw_on(int rc) {
    if (rc == FHT_OK) return;
    const std::string msg = fht_last_error();
    if (rc == FHT_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == FHT_ERR_OVERFLOW) throw std::overflow_error(msg);
    if (rc == FHT_ERR_NOMEM) throw std::bad_alloc();
    throw std::runtime_error("fht_b200: " + msg);
}

// ------------------------------------------------------------------ image
using Accum = std::int64_t;

class Image {
public:
    Image() = default;
    Image(int width, int height)
        : w_(checked_width(width, height)), h_(height),
          data_(static_cast<std::size_t>(width) * static_cast<std::size_t>(height), 0) {}
    Image(int width, int height, std::vector<Accum> data)
        : w_(checked_width(width, height)), h_(height), data_(std::move(data)) {
        if (data_.size() != static_cast<std::size_t>(w_) * static_cast<std::size_t>(h_))
            throw std::invalid_argument("Image: data length does not equal width*height");
    }
    int width() const { return w_; }
    int height() const { return h_; }
    bool empty() const { return data_.empty(); }
    Accum operator()(int x, int y) const { return data_[index(x, y)]; }
    Accum& operator()(int x, int y) { return data_[index(x, y)]; }
    std::span<const Accum> row(int y) const { return {data_.data() + index(0, y), static_cast<std::size_t>(w_)}; }
    std::span<Accum> row(int y) { return {data_.data() + index(0, y), static_cast<std::size_t>(w_)}; }
    const std::vector<Accum>& data() const { return data_; }
    std::vector<Accum>& data() { return data_; }
    bool operator==(const Image&) const = default;

private:
    static int checked_width(int w, int h) {
        if (w < 1 || h < 1) throw std::invalid_argument("Image: width and height must be positive");
        return w;
    }
    std::size_t index(int x, int y) const {
        return static_cast<std::size_t>(y) * static_cast<std::size_t>(w_) + static_cast<std::size_t>(x);
    }
    int w_ = 0;
    int h_ = 0;
    std::vector<Accum> data_;
};

using HoughImage = Image;

// ------------------------------------------------------------ split rules
enum class SplitStrategy { Simple, Tweaked };

inline const char* to_string(SplitStrategy s) { return s == SplitStrategy::Simple ? "simple" : "tweaked"; }

inline SplitStrategy strategy_from_string(const std::string& name) {
    if (name == "simple") return SplitStrategy::Simple;
    if (name == "tweaked") return SplitStrategy::Tweaked;
    throw std::invalid_argument("unknown strategy '" + name + "' (expected simple|tweaked)");
}

inline int strategy_code(SplitStrategy s) { return s == SplitStrategy::Simple ? FHT_SPLIT_SIMPLE : FHT_SPLIT_TWEAKED; }

inline int floor_log2(std::int64_t n) {
    if (n < 1) throw std::invalid_argument("floor_log2: argument must be positive");
    return std::bit_width(static_cast<std::uint64_t>(n)) - 1;
}

inline std::pair<int, int> split_width(int w, SplitStrategy strategy) {
    int a = 0, b = 0;
    throw_on(fht_split_width(w, strategy_code(strategy), &a, &b));
    return {a, b};
}
inline std::pair<int, int> split_simple(int w) { return split_width(w, SplitStrategy::Simple); }
inline std::pair<int, int> split_tweaked(int w) { return split_width(w, SplitStrategy::Tweaked); }

inline std::int64_t round_half_up_ratio(std::int64_t num, std::int64_t den) {
    std::int64_t r = 0;
    throw_on(fht_round_half_up_ratio(num, den, &r));
    return r;
}

// --------------------------------------------------------------- transform
/// Circular shift u(i) = v((i + r) mod h), r in [0, h) (transform.cpp:8-14).
inline std::vector<Accum> rotate(std::span<const Accum> v, int r) {
    const int h = static_cast<int>(v.size());
    if (r < 0 || r >= h) throw std::invalid_argument("rotate: shift must lie in [0, h)");
    std::vector<Accum> out(v.size());
    for (int i = 0; i < h; ++i) out[static_cast<std::size_t>(i)] = v[static_cast<std::size_t>((i + r) % h)];
    return out;
}

/// width * max|value| < 2^62, else std::overflow_error (transform.cpp:16-27).
inline void check_overflow_budget(const Image& img) {
    std::uint64_t vmax = 0;
    for (const Accum v : img.data()) {
        const std::uint64_t a = v < 0 ? 0u - static_cast<std::uint64_t>(v) : static_cast<std::uint64_t>(v);
        vmax = a > vmax ? a : vmax;
    }
    if (static_cast<unsigned __int128>(img.width()) * vmax >= (static_cast<unsigned __int128>(1) << 62))
        throw std::overflow_error("fht2d: width * max|value| reaches 2^62; sums could overflow 64-bit accumulators");
}

struct CountedTransform {
    HoughImage hough;
    std::uint64_t additions = 0;
};

inline CountedTransform fht2d_counted(const Image& img, SplitStrategy strategy) {
    if (img.empty()) throw std::invalid_argument("fht2d: image is empty");
    CountedTransform r{HoughImage(img.width(), img.height()), 0};
    throw_on(fht_fht2d_counted_i64(img.data().data(), img.width(), img.height(), strategy_code(strategy),
                                   r.hough.data().data(), &r.additions));
    return r;
}

inline HoughImage fht2d(const Image& img, SplitStrategy strategy) { return fht2d_counted(img, strategy).hough; }

// --------------------------------------------------------------- quadrants
inline Image flip_horizontal(const Image& img) {
    Image out(img.width(), img.height());
    for (int y = 0; y < img.height(); ++y)
        for (int x = 0; x < img.width(); ++x) out(x, y) = img(img.width() - 1 - x, y);
    return out;
}

inline Image transpose(const Image& img) {
    Image out(img.height(), img.width());
    for (int y = 0; y < img.height(); ++y)
        for (int x = 0; x < img.width(); ++x) out(y, x) = img(x, y);
    return out;
}

struct QuadrantSet {
    HoughImage horiz_pos;
    HoughImage horiz_neg;
    HoughImage vert_pos;
    HoughImage vert_neg;
};

/// All four families in one device call; the flips and transposes are index
/// maps inside the kernels, not copies.
inline QuadrantSet fht2d_quadrants(const Image& img, SplitStrategy strategy,
                                   std::uint64_t* total_additions = nullptr) {
    if (img.empty()) throw std::invalid_argument("fht2d: image is empty");
    const int w = img.width(), h = img.height();
    QuadrantSet q{HoughImage(w, h), HoughImage(w, h), HoughImage(h, w), HoughImage(h, w)};
    std::uint64_t adds = 0;
    throw_on(fht_fht2d_quadrants_i64(img.data().data(), w, h, strategy_code(strategy), q.horiz_pos.data().data(),
                                     q.horiz_neg.data().data(), q.vert_pos.data().data(), q.vert_neg.data().data(),
                                     &adds));
    if (total_additions) *total_additions = adds;
    return q;
}

// ------------------------------------------------------ patterns / oracle
/// pattern.hpp:12-17
struct Pattern {
    int n = 0;
    int t = 0;
    std::vector<int> values;
};

/// Algorithm 2 (pattern.cpp:24-30).
inline Pattern fht2d_pattern(int n, int t, SplitStrategy strategy) {
    Pattern p{n, t, std::vector<int>(n > 0 ? static_cast<std::size_t>(n) : 0)};
    throw_on(fht_fht2d_pattern(n, t, strategy_code(strategy), p.values.data()));
    return p;
}

/// pattern.cpp:32-38
inline std::vector<Pattern> pattern_set(int n, SplitStrategy strategy) {
    if (n < 1) throw std::invalid_argument("pattern_set: width must be positive");
    std::vector<Pattern> set;
    set.reserve(static_cast<std::size_t>(n));
    for (int t = 0; t < n; ++t) set.push_back(fht2d_pattern(n, t, strategy));
    return set;
}

/// oracle.cpp:9-25: direct summation along every shifted pattern (on the GPU).
inline HoughImage slow_hough(const Image& img, SplitStrategy strategy) {
    if (img.empty()) throw std::invalid_argument("slow_hough: image is empty");
    HoughImage out(img.width(), img.height());
    throw_on(fht_slow_hough_i64(img.data().data(), img.width(), img.height(), strategy_code(strategy),
                                out.data().data()));
    return out;
}

/// oracle.cpp:27-33
inline std::uint64_t count_additions_tree(int w, int h, SplitStrategy strategy) {
    std::uint64_t r = 0;
    throw_on(fht_count_additions_tree(w, h, strategy_code(strategy), &r));
    return r;
}

// --------------------------------------------------------- batched plans
/// RAII owner of an fht_plan_t: device-resident batched execution.
class Plan {
public:
    Plan(int width, int height, SplitStrategy strategy, int in_dtype, int acc_dtype, int out_dtype,
         int quadrant_mask = FHT_ALL_QUADRANTS, int batch = 1, int layout = FHT_LAYOUT_REFERENCE, int device = 0) {
        throw_on(fht_plan_create(width, height, strategy_code(strategy), in_dtype, acc_dtype, out_dtype, quadrant_mask,
                                 batch, layout, device, &p_));
    }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    Plan(Plan&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
    ~Plan() {
        if (p_) fht_plan_destroy(p_);
    }
    std::size_t workspace_bytes() const { return fht_workspace_bytes(p_); }
    std::uint64_t additions() const { return fht_additions(p_); }
    int launches_per_execute() const { return fht_launches_per_execute(p_); }
    void execute(const void* d_in, std::int64_t in_stride, void* const d_out[4], std::int64_t out_stride,
                 void* d_workspace, void* stream = nullptr) const {
        throw_on(fht_execute(p_, d_in, in_stride, d_out, out_stride, d_workspace, stream));
    }
    void execute_host(const void* h_in, void* const h_out[4], void* stream = nullptr) const {
        throw_on(fht_execute_host(p_, h_in, h_out, stream));
    }
    fht_plan_t get() const { return p_; }

private:
    fht_plan_t p_ = nullptr;
};

}  // namespace fht_b200
