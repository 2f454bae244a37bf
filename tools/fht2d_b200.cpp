// fht2d_b200 -- the reference CLI's transform path on the GPU.
//
// Mirrors `fht2d transform` / `pattern` / `analyze` of the reference CLI
// (tools/fht2d_main.cpp:52-108, 112-175) with the same options, file formats
// and exit behaviour:
//   fht2d_b200 transform --input a.pgm --strategy simple|tweaked --output j.fht1|j.csv
//                        [--count] [--quadrants]
//   fht2d_b200 pattern --n N --t T --strategy simple|tweaked
//   fht2d_b200 analyze complexity|error --n-max N [--fast] --output OUT.csv
// Input: PGM P2/P5, maxval <= 65535, w*h <= 2^30 (pgm.cpp:42-87).  Output: the
// FHT1 raster (magic "FHT1", u32 LE width/height, dtype byte 0, int64 LE
// payload, x fastest; raster.hpp:10-19) or, for a .csv path, one line per shift
// s (fht2d_main.cpp:32-43).  --quadrants writes <output>.{hpos,hneg,vpos,vneg}
// (fht2d_main.cpp:22-29).  Errors: "fht2d: <what>" on stderr, exit 1.
//
// The image goes to the device as 8- or 16-bit samples (not widened to int64
// on the host); the transform accumulates in int32 when width * maxval < 2^31
// (always for 8-bit input below 8.4M columns) and int64 otherwise, and the
// root pass widens to int64 on the device.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fht_b200.h"

namespace {

[[noreturn]] void fail(const std::string& what) { throw std::runtime_error(what); }

void check(int rc) {
    if (rc != FHT_OK) throw std::runtime_error(fht_last_error());
}

// ---------------------------------------------------------------- PGM input
struct Pgm {
    int w = 0, h = 0;
    long maxval = 0;
    std::vector<uint16_t> samples;  // row-major, x fastest
};

long header_number(std::istream& in, const char* what) {
    int c = in.get();
    for (;;) {  // whitespace and '#' comments to end of line
        if (c == '#') {
            while (c != '\n' && c != EOF) c = in.get();
        } else if (c != EOF && std::isspace(c)) {
            c = in.get();
        } else {
            break;
        }
    }
    if (c == EOF) fail(std::string("pgm: unexpected end of file before ") + what);
    if (c < '0' || c > '9') fail(std::string("pgm: malformed ") + what);
    long v = 0;
    while (c >= '0' && c <= '9') {
        v = v * 10 + (c - '0');
        if (v > 1000000000L) fail(std::string("pgm: ") + what + " out of range");
        c = in.get();
    }
    if (c != EOF) in.unget();
    return v;
}

Pgm read_pgm(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail("pgm: cannot open '" + path + "'");
    char magic[2] = {0, 0};
    in.read(magic, 2);
    if (!in || magic[0] != 'P' || (magic[1] != '2' && magic[1] != '5'))
        fail("pgm: not a PGM file (expected P2 or P5 magic)");
    const bool binary = magic[1] == '5';
    Pgm p;
    const long w = header_number(in, "width"), h = header_number(in, "height");
    p.maxval = header_number(in, "maxval");
    if (w < 1 || h < 1) fail("pgm: width and height must be positive");
    if (w * h > (1L << 30)) fail("pgm: image too large");
    if (p.maxval < 1 || p.maxval > 65535) fail("pgm: unsupported maxval " + std::to_string(p.maxval));
    p.w = static_cast<int>(w);
    p.h = static_cast<int>(h);
    const size_t n = static_cast<size_t>(w) * static_cast<size_t>(h);
    p.samples.resize(n);
    if (binary) {
        const int c = in.get();  // one whitespace byte before the raster
        if (c == EOF || !std::isspace(c)) fail("pgm: missing whitespace before binary raster");
        const int bps = p.maxval > 255 ? 2 : 1;
        std::vector<unsigned char> raw(n * static_cast<size_t>(bps));
        in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
        if (in.gcount() != static_cast<std::streamsize>(raw.size())) fail("pgm: truncated raster payload");
        for (size_t i = 0; i < n; ++i) {
            const long v = bps == 1 ? raw[i] : raw[2 * i] * 256L + raw[2 * i + 1];  // 16-bit: big-endian
            if (v > p.maxval) fail("pgm: sample exceeds maxval");
            p.samples[i] = static_cast<uint16_t>(v);
        }
    } else {
        for (size_t i = 0; i < n; ++i) {
            const long v = header_number(in, "sample");
            if (v > p.maxval) fail("pgm: sample exceeds maxval");
            p.samples[i] = static_cast<uint16_t>(v);
        }
    }
    return p;
}

// ----------------------------------------------------------------- output
bool ends_with(const std::string& s, const std::string& suf) {
    return s.size() >= suf.size() && s.compare(s.size() - suf.size(), suf.size(), suf) == 0;
}

// "dir/out.fht1" + "hpos" -> "dir/out.hpos.fht1"; no extension -> "out.hpos"
std::string suffixed(const std::string& path, const std::string& tag) {
    const size_t slash = path.find_last_of('/'), dot = path.find_last_of('.');
    if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) return path + "." + tag;
    return path.substr(0, dot) + "." + tag + path.substr(dot);
}

void write_output(const std::string& path, const int64_t* j, int w, int h) {
    if (ends_with(path, ".csv")) {
        std::ofstream out(path, std::ios::trunc);
        if (!out) fail("cannot open '" + path + "' for writing");
        std::string line;
        for (int s = 0; s < h; ++s) {
            line.clear();
            for (int t = 0; t < w; ++t) {
                if (t) line += ',';
                line += std::to_string(j[static_cast<size_t>(s) * w + t]);
            }
            line += '\n';
            out << line;
        }
        if (!out) fail("write failed for '" + path + "'");
        return;
    }
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail("raster: cannot open '" + path + "' for writing");
    unsigned char hdr[13] = {'F', 'H', 'T', '1'};
    for (int i = 0; i < 4; ++i) {
        hdr[4 + i] = static_cast<unsigned char>((static_cast<uint32_t>(w) >> (8 * i)) & 0xff);
        hdr[8 + i] = static_cast<unsigned char>((static_cast<uint32_t>(h) >> (8 * i)) & 0xff);
    }
    hdr[12] = 0;  // dtype: signed 64-bit
    out.write(reinterpret_cast<const char*>(hdr), 13);
    const size_t n = static_cast<size_t>(w) * h;
    std::vector<unsigned char> buf(n * 8);
    for (size_t i = 0; i < n; ++i) {
        const uint64_t u = static_cast<uint64_t>(j[i]);
        for (int b = 0; b < 8; ++b) buf[i * 8 + static_cast<size_t>(b)] = static_cast<unsigned char>((u >> (8 * b)) & 0xff);
    }
    out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
    if (!out) fail("raster: write failed");
}

// ------------------------------------------------------------------ runs
int strategy_of(const std::string& s) {
    if (s == "simple") return FHT_SPLIT_SIMPLE;
    if (s == "tweaked") return FHT_SPLIT_TWEAKED;
    fail("unknown strategy '" + s + "' (expected simple|tweaked)");
}

int run_transform(const std::string& input, const std::string& output, int strategy, bool count, bool quadrants) {
    const Pgm p = read_pgm(input);
    const int mask = quadrants ? FHT_ALL_QUADRANTS : FHT_HORIZ_POS;
    const int64_t wmax = quadrants ? std::max(p.w, p.h) : p.w;
    const bool eight = p.maxval <= 255;
    const int in_dt = eight ? FHT_U8 : FHT_I32;
    const int acc = wmax * p.maxval < (int64_t(1) << 31) ? FHT_I32 : FHT_I64;
    fht_plan_t plan = nullptr;
    check(fht_plan_create(p.w, p.h, strategy, in_dt, acc, FHT_I64, mask, 1, FHT_LAYOUT_REFERENCE, 0, &plan));
    const size_t n = static_cast<size_t>(p.w) * p.h;
    std::vector<uint8_t> in8;
    std::vector<int32_t> in32;
    const void* h_in;
    if (eight) {
        in8.assign(p.samples.begin(), p.samples.end());
        h_in = in8.data();
    } else {
        in32.assign(p.samples.begin(), p.samples.end());
        h_in = in32.data();
    }
    std::vector<int64_t> outs[4];
    void* ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int q = 0; q < 4; ++q)
        if (mask & (1 << q)) {
            outs[q].resize(n);
            ptrs[q] = outs[q].data();
        }
    const int rc = fht_execute_host(plan, h_in, ptrs, nullptr);
    const uint64_t additions = fht_additions(plan);
    fht_plan_destroy(plan);
    check(rc);
    if (quadrants) {
        static const char* tags[4] = {"hpos", "hneg", "vpos", "vneg"};
        for (int q = 0; q < 4; ++q) {
            const int W = q < 2 ? p.w : p.h, H = q < 2 ? p.h : p.w;
            write_output(suffixed(output, tags[q]), outs[q].data(), W, H);
        }
    } else {
        write_output(output, outs[0].data(), p.w, p.h);
    }
    if (count) std::cout << additions << "\n";
    return 0;
}

int run_pattern(int n, int t, int strategy) {
    if (n < 1) fail("--n must be positive");
    std::vector<int> v(static_cast<size_t>(n));
    check(fht_fht2d_pattern(n, t, strategy, v.data()));
    for (int x = 0; x < n; ++x) std::cout << (x ? "," : "") << v[static_cast<size_t>(x)];
    std::cout << "\n";
    return 0;
}

// ---------------------------------------------------------------- analyze
// fht2d_main.cpp:81-108 with the csv.cpp layouts; the Theta(n^3) error sweep
// runs on the GPU (fht_max_deviation_numerators).
std::string sig(double v) {  // csv.cpp:10-16: 12 significant digits, general format
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.12g", v);
    return buf;
}

int floor_log2i(int64_t n) {
    int q = 0;
    while ((int64_t(1) << (q + 1)) <= n) ++q;
    return q;
}

int run_analyze(const std::string& mode, int n_max, bool fast, const std::string& output) {
    if (n_max < 1) fail("--n-max must be positive");
    std::ofstream out(output, std::ios::trunc);
    if (!out) fail("cannot open '" + output + "' for writing");
    if (mode == "complexity") {
        out << "n,f_simple,f_tweaked,norm_simple,norm_tweaked\n";
        for (int n = 1; n <= n_max; ++n) {
            uint64_t fs = 0, ft = 0;
            check(fht_count_additions_tree(n, n, FHT_SPLIT_SIMPLE, &fs));
            check(fht_count_additions_tree(n, n, FHT_SPLIT_TWEAKED, &ft));
            out << n << ',' << fs << ',' << ft << ',';
            if (n > 1) {
                const double d = static_cast<double>(n) * static_cast<double>(n) * std::log2(static_cast<double>(n));
                out << sig(static_cast<double>(fs) / d) << ',' << sig(static_cast<double>(ft) / d);
            } else {
                out << ',';
            }
            out << '\n';
        }
    } else if (mode == "error") {
        std::vector<int> sizes;
        for (int n = 1; n <= (fast ? std::min(n_max, 1024) : n_max); ++n) sizes.push_back(n);
        if (fast)
            for (int s : {1451, 2048, 4095, 4096})
                if (s <= n_max) sizes.push_back(s);
        const int lo = 1, hi = fast ? std::min(n_max, 1024) : n_max;
        std::vector<int64_t> ws(static_cast<size_t>(hi)), wt(static_cast<size_t>(hi));
        check(fht_max_deviation_numerators(lo, hi, FHT_SPLIT_SIMPLE, ws.data()));
        check(fht_max_deviation_numerators(lo, hi, FHT_SPLIT_TWEAKED, wt.data()));
        out << "n,e_simple,e_tweaked,bound,norm_simple,norm_tweaked\n";
        int64_t exceeding = 0;
        for (int n : sizes) {
            int64_t a = 0, b = 0;
            if (n <= hi) {
                a = ws[static_cast<size_t>(n - 1)];
                b = wt[static_cast<size_t>(n - 1)];
            } else {
                check(fht_max_deviation_numerators(n, n, FHT_SPLIT_SIMPLE, &a));
                check(fht_max_deviation_numerators(n, n, FHT_SPLIT_TWEAKED, &b));
            }
            const int64_t den = n == 1 ? 1 : n - 1;
            const int q = floor_log2i(n);
            const int64_t p = int64_t(1) << q, bnum = q * p + 6 * p - 6, bden = 6 * p;  // analysis.cpp:23-28
            const double es = static_cast<double>(a) / static_cast<double>(den);
            const double et = static_cast<double>(b) / static_cast<double>(den);
            out << n << ',' << sig(es) << ',' << sig(et) << ',' << sig(static_cast<double>(bnum) / static_cast<double>(bden))
                << ',';
            if (n > 1) {
                const double sc = 6.0 / std::log2(static_cast<double>(n));
                out << sig(es * sc) << ',' << sig(et * sc);
            } else {
                out << ',';
            }
            out << '\n';
            // e_simple > bound, exactly: a / den > bnum / bden
            if (static_cast<__int128>(a) * bden > static_cast<__int128>(bnum) * den) ++exceeding;
        }
        std::cout << sig(static_cast<double>(exceeding) / static_cast<double>(sizes.size())) << "\n";
    } else {
        fail("unknown analyze mode '" + mode + "' (expected complexity|error)");
    }
    if (!out) fail("write failed for '" + output + "'");
    return 0;
}

void usage() {
    std::cerr << "usage: fht2d_b200 transform --input IMG.pgm --strategy simple|tweaked --output OUT[.csv]"
                 " [--count] [--quadrants]\n"
                 "       fht2d_b200 pattern --n N --t T --strategy simple|tweaked\n"
                 "       fht2d_b200 analyze complexity|error --n-max N [--fast] --output OUT.csv\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 1;
    }
    const std::string cmd = argv[1];
    std::string input, output, strategy;
    bool count = false, quadrants = false, have_n = false, have_t = false, fast = false;
    int n = 0, t = 0, n_max = 0;
    std::string mode;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto value = [&]() -> std::string {
                if (i + 1 >= argc) fail(a + " requires a value");
                return argv[++i];
            };
            if (a == "--input") input = value();
            else if (a == "--output") output = value();
            else if (a == "--strategy") strategy = value();
            else if (a == "--count") count = true;
            else if (a == "--quadrants") quadrants = true;
            else if (a == "--n") n = std::stoi(value()), have_n = true;
            else if (a == "--t") t = std::stoi(value()), have_t = true;
            else if (a == "--n-max") n_max = std::stoi(value());
            else if (a == "--fast") fast = true;
            else if (cmd == "analyze" && mode.empty() && a.rfind("--", 0) != 0) mode = a;
            else if (a == "-h" || a == "--help") {
                usage();
                return 0;
            } else {
                fail("unknown option " + a);
            }
        }
        if (cmd == "transform") {
            if (input.empty() || output.empty() || strategy.empty())
                fail("transform requires --input, --strategy and --output");
            return run_transform(input, output, strategy_of(strategy), count, quadrants);
        }
        if (cmd == "pattern") {
            if (!have_n || !have_t || strategy.empty()) fail("pattern requires --n, --t and --strategy");
            return run_pattern(n, t, strategy_of(strategy));
        }
        if (cmd == "analyze") {
            if (mode.empty() || output.empty()) fail("analyze requires a mode, --n-max and --output");
            return run_analyze(mode, n_max, fast, output);
        }
        fail("unknown subcommand '" + cmd + "' (expected transform|pattern|analyze)");
    } catch (const std::exception& e) {
        std::cerr << "fht2d: " << e.what() << "\n";
        return 1;
    }
}
