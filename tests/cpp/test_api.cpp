// C++ drop-in test: reference-style code (namespace fht via as_fht.hpp)
// against libfht_b200.so, checked against the oracle's C restatement
// (oracle/liboracle.so, test infrastructure).  Built and run by
// tests/test_cpp_api.py on a GPU box.
#include <cstdint>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "fht_b200/as_fht.hpp"

extern "C" int oracle_fht2d_counted(const int64_t*, int, int, int, int64_t*, uint64_t*);
extern "C" int oracle_fht2d_quadrants_i64(const int64_t*, int, int, int, int64_t*, int64_t*, int64_t*, int64_t*,
                                          uint64_t*);

static int failures = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                 \
        }                                                               \
    } while (0)

int main() {
    // SPEC.md:93 2x2 example: I(0,0)=a I(1,0)=b I(0,1)=c I(1,1)=d
    fht::Image two(2, 2, {3, 5, 7, 11});
    fht::HoughImage j = fht::fht2d(two, fht::SplitStrategy::Tweaked);
    CHECK(j(0, 0) == 3 + 5 && j(0, 1) == 7 + 11 && j(1, 0) == 3 + 11 && j(1, 1) == 7 + 5);

    CHECK(fht::split_tweaked(17) == std::make_pair(16, 1));
    CHECK(fht::split_simple(17) == std::make_pair(8, 9));
    CHECK(fht::round_half_up_ratio(1, 2) == 1);
    CHECK(fht::strategy_from_string("simple") == fht::SplitStrategy::Simple);

    std::mt19937_64 rng(7);
    std::uniform_int_distribution<int64_t> dist(-100000, 100000);
    for (auto [w, h] : {std::pair{1, 1}, {1, 9}, {9, 1}, {17, 17}, {37, 23}, {23, 37}, {100, 33}, {509, 64}}) {
        for (auto s : {fht::SplitStrategy::Simple, fht::SplitStrategy::Tweaked}) {
            fht::Image img(w, h);
            for (auto& v : img.data()) v = dist(rng);
            fht::CountedTransform ct = fht::fht2d_counted(img, s);
            std::vector<int64_t> ref(static_cast<size_t>(w) * h);
            uint64_t adds = 0;
            CHECK(oracle_fht2d_counted(img.data().data(), w, h, s == fht::SplitStrategy::Simple ? 0 : 1, ref.data(),
                                       &adds) == 0);
            CHECK(ct.hough.data() == ref);
            CHECK(ct.additions == adds);
            uint64_t qadds = 0, radds = 0;
            fht::QuadrantSet q = fht::fht2d_quadrants(img, s, &qadds);
            std::vector<int64_t> r0(ref.size()), r1(ref.size()), r2(ref.size()), r3(ref.size());
            CHECK(oracle_fht2d_quadrants_i64(img.data().data(), w, h, s == fht::SplitStrategy::Simple ? 0 : 1, r0.data(),
                                             r1.data(), r2.data(), r3.data(), &radds) == 0);
            CHECK(q.horiz_pos.data() == r0 && q.horiz_neg.data() == r1 && q.vert_pos.data() == r2 &&
                  q.vert_neg.data() == r3);
            CHECK(qadds == radds);
            CHECK(q.vert_pos.width() == h && q.vert_pos.height() == w);
        }
    }
    // exception types mirror the reference (transform.cpp:24-26, 63)
    bool threw = false;
    try {
        fht::fht2d(fht::Image(), fht::SplitStrategy::Tweaked);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        fht::Image big(4, 2);
        for (auto& v : big.data()) v = int64_t(1) << 61;
        fht::fht2d(big, fht::SplitStrategy::Tweaked);
    } catch (const std::overflow_error&) {
        threw = true;
    }
    CHECK(threw);
    // batched plan, u8 -> i32 through the RAII wrapper
    {
        fht::Plan plan(64, 48, fht::SplitStrategy::Tweaked, FHT_U8, FHT_I32, FHT_I32, FHT_ALL_QUADRANTS, 2);
        uint64_t ch = 0, cv = 0;
        CHECK(fht_count_additions_tree(64, 48, FHT_SPLIT_TWEAKED, &ch) == FHT_OK);
        CHECK(fht_count_additions_tree(48, 64, FHT_SPLIT_TWEAKED, &cv) == FHT_OK);
        CHECK(plan.additions() == 2 * (2 * ch + 2 * cv));
        std::vector<uint8_t> in(2 * 64 * 48);
        for (auto& v : in) v = static_cast<uint8_t>(rng() & 255);
        std::vector<int32_t> out[4];
        void* ptrs[4];
        for (int k = 0; k < 4; ++k) {
            out[k].resize(in.size());
            ptrs[k] = out[k].data();
        }
        plan.execute_host(in.data(), ptrs);
        fht::Image img(64, 48);
        for (size_t i = 0; i < img.data().size(); ++i) img.data()[i] = in[64 * 48 + i];
        fht::QuadrantSet q = fht::fht2d_quadrants(img, fht::SplitStrategy::Tweaked);
        for (size_t i = 0; i < img.data().size(); ++i) CHECK(out[2][64 * 48 + i] == q.vert_pos.data()[i]);
    }
    // patterns and the structure-free oracle (pattern.cpp, oracle.cpp)
    CHECK(fht::fht2d_pattern(4, 1, fht::SplitStrategy::Tweaked).values == std::vector<int>({0, 0, 1, 1}));
    CHECK(fht::pattern_set(4, fht::SplitStrategy::Tweaked)[2].values == std::vector<int>({0, 1, 1, 2}));
    CHECK(fht::count_additions_tree(17, 17, fht::SplitStrategy::Tweaked) == 1377);
    {
        fht::Image img(45, 31);
        for (auto& v : img.data()) v = dist(rng);
        CHECK(fht::slow_hough(img, fht::SplitStrategy::Simple) == fht::fht2d(img, fht::SplitStrategy::Simple));
    }
    std::printf("%s (%d failures)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
