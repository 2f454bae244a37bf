// capi.cu -- the extern "C" boundary (include/fht_b200.h) over the plan
// tables (plan.cpp) and the sm_100a kernels (kernels.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <cstdint>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fht_b200.h"
#include "kernels.cuh"
#include "plan.hpp"
#include "slow.cuh"

using fhtb::GroupLaunch;
using fhtb::QuadSet;
using fhtb::ShapeHdr;
using fhtb::SubPlan;

namespace {

thread_local std::string g_last_error;

struct FhtError : std::runtime_error {
    int code;
    FhtError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Host synchronisations and device allocations the library makes (for the
// tests that check a timed step does neither: fht_debug_counters).
std::atomic<unsigned long long> g_host_syncs{0}, g_device_allocs{0};
cudaError_t counted_sync(cudaStream_t s) {
    g_host_syncs.fetch_add(1, std::memory_order_relaxed);
    return cudaStreamSynchronize(s);
}
template <class T>
cudaError_t counted_malloc(T** p, size_t n) {
    g_device_allocs.fetch_add(1, std::memory_order_relaxed);
    return cudaMalloc(p, n);
}
template <class T>
cudaError_t counted_malloc_async(T** p, size_t n, cudaStream_t s) {
    g_device_allocs.fetch_add(1, std::memory_order_relaxed);
    return cudaMallocAsync(p, n, s);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw FhtError(FHT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FHT_OK;
    } catch (const FhtError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return FHT_ERR_INVALID;
    } catch (const std::overflow_error& e) {
        g_last_error = e.what();
        return FHT_ERR_OVERFLOW;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return FHT_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FHT_ERR_INTERNAL;
    }
}

size_t esize(int dt) {
    switch (dt) {
        case FHT_U8: return 1;
        case FHT_I32: return 4;
        case FHT_I64: return 8;
        case FHT_F32: return 4;
    }
    throw FhtError(FHT_ERR_INVALID, "unknown dtype");
}

bool valid_types(int in, int acc, int out) {
    if (acc == FHT_I32 && out == FHT_I32) return in == FHT_U8 || in == FHT_I32;
    if (acc == FHT_I32 && out == FHT_I64) return in == FHT_U8 || in == FHT_I32 || in == FHT_I64;
    if (acc == FHT_I64 && out == FHT_I64) return in == FHT_U8 || in == FHT_I32 || in == FHT_I64;
    if (acc == FHT_F32 && out == FHT_F32) return in == FHT_F32 || in == FHT_U8;
    return false;
}

// Device copy of one SubPlan's tables in a single allocation.
struct DevTables {
    void* blob = nullptr;
    const int4* blocks = nullptr;
    const int* by_x0 = nullptr;
    const ShapeHdr* shapes = nullptr;
    const int* step_offs = nullptr;
    const fhtb::PassOpDev* k1_ops = nullptr;
    const int4* k1_bops = nullptr;
    std::vector<fhtb::PassDev> passes;  // device pointers; S/L filled by create_plan
    int max_ops = 0, max_steps = 0;
};

struct Group {
    QuadSet qs{};
    SubPlan sp;
    DevTables dt;
    int ld = 0, S = 0, sr = 0, nbuf = 0;
    int nblocks = 0, nby = 0;
    bool use_by32 = false;
    bool pairs = false;  // K2 runs the level-pair programs (4-byte accumulators)
    // u8 staging for K1P (kernels.cuh GroupLaunch::stage): bytes per image,
    // column pitch, offsets of the T / P column sets (-1: not staged)
    long long stage_img = 0, stage_pitch = 0, stage_t = -1, stage_p = -1;
    std::vector<int> pass_S, pass_L;  // K2 rows per tile and slot capacity, per pass
    int pm_D = 0;  // u16 pair mode (0: off): workspace words pair rows j and j + pm_D
    bool k1_acc32 = false;  // int64 plan, pass 0 in int32 (GroupLaunch::k1_acc32)
    size_t slot_bytes = 0;
    size_t acc_sz = 4;  // accumulator bytes
};

int round_up(int v, int m) { return (v + m - 1) / m * m; }

bool esize_acc4(const Group& g) { return g.acc_sz == 4; }

constexpr int kHostStreams = 3;

int env_int(const char* name, int def, int lo, int hi) {
    if (const char* e = std::getenv(name)) return std::max(lo, std::min(hi, std::atoi(e)));
    return def;
}

// The tile program K2 executes for a pass: one level per step (PassOp), or
// the level-pair program (PassOpN, plan.hpp) -- same tiles and loads.
struct PassProgram {
    const std::vector<fhtb::PassTile>& tiles;
    const std::vector<int>& step_offs;
    const std::vector<fhtb::PassStore>& stores;
    int max_slots;
    int max_tile_ops() const {
        int m = 0;
        for (const auto& t : tiles)
            m = std::max(m, step_offs[static_cast<size_t>(t.step_beg + t.nsteps)] - step_offs[static_cast<size_t>(t.step_beg)]);
        return m;
    }
};
PassProgram program(const fhtb::FusedPass& ps, bool pairs) {
    if (pairs) return {ps.ptiles, ps.pstep_offs, ps.pstores, ps.pmax_slots};
    return {ps.tiles, ps.step_offs, ps.stores, ps.max_slots};
}


}  // namespace

struct fht_plan_s {
    int w = 0, h = 0, strategy = 1, in = 0, acc = 1, out = 1, mask = 15, batch = 1, layout = 0, device = 0;
    std::vector<std::unique_ptr<Group>> groups;
    int chunk = 1;
    int num_sms = 148;
    size_t ws_bytes = 0;
    size_t slot_bytes_img = 0, stage_bytes_img = 0;  // workspace per image: slot buffers, then u8 staging
    int launches = 0;
    uint64_t additions = 0;
    std::mutex host_mu;
    void* st_in = nullptr;
    void* st_out[4] = {nullptr, nullptr, nullptr, nullptr};
    void* st_ws = nullptr;
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::mutex fork_mu;  // serialises each ev_fork/ev_join record + wait pair (kernels.cu launch_typed)
    cudaStream_t hst[kHostStreams] = {};  // execute_host pipeline
    cudaEvent_t hev[kHostStreams] = {};
    cudaEvent_t hev_start = nullptr;

    ~fht_plan_s() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (aux) cudaStreamDestroy(aux);
        for (int k = 0; k < kHostStreams; ++k) {
            if (hst[k]) cudaStreamDestroy(hst[k]);
            if (hev[k]) cudaEventDestroy(hev[k]);
        }
        if (hev_start) cudaEventDestroy(hev_start);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        for (auto& g : groups)
            if (g->dt.blob) cudaFree(g->dt.blob);
        if (st_in) cudaFree(st_in);
        for (void* p : st_out)
            if (p) cudaFree(p);
        if (st_ws) cudaFree(st_ws);
        cudaSetDevice(prev);
    }
};

namespace {

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// One K2 window as copies for the TMA engine (k2_pair_pipe, FHT_K2_TMA):
// rows (start + i) mod H, i < n, of a column (ld words allocated) into a
// shared slot.  The window is placed at word `delta` of its slot so that the
// long piece is a 16-byte aligned bulk copy (cp.async.bulk); the rest (the
// part of a wrapping window whose alignment differs by H mod 4, and the <= 3
// words before H rounded down) goes by 4-byte cp.async.  All word offsets.
struct WinCopy {
    int delta = 0, bulk_src = 0, bulk_dst = 0, bulk_words = 0, small_src = 0, small_dst = 0, small_n = 0;
    bool ok = true;
};
WinCopy window_copy(int off, int n, int H, int ld) {
    WinCopy c;
    const int start = ((off % H) + H) % H;
    if (n > H) {  // a window longer than the column (tiny H): all small copies
        c.ok = false;
        return c;
    }
    if (start + n <= H) {  // no wrap: one bulk copy (rounded up into the slot's slack)
        c.delta = start & 3;
        c.bulk_src = start - c.delta;
        c.bulk_words = (n + c.delta + 3) & ~3;
        c.ok = c.bulk_src + c.bulk_words <= ld;
        return c;
    }
    const int a = H - start, b = n - a;  // [start, H) then [0, b)
    const int h_al = H & ~3;
    const int c1 = std::max(0, h_al - start);  // option 1: piece A in bulk up to H rounded down
    if (n - c1 <= a) {
        c.delta = start & 3;
        if (c1 > 0) {
            c.bulk_src = start - c.delta;
            c.bulk_words = c1 + c.delta;
        }
        c.small_src = start + c1;  // wraps mod H in the kernel
        c.small_dst = c.delta + c1;
        c.small_n = n - c1;
    } else {  // option 2: piece B in bulk (aligned at word 0), piece A small
        c.delta = (4 - (a & 3)) & 3;
        c.bulk_src = 0;
        c.bulk_dst = c.delta + a;
        c.bulk_words = (b + 3) & ~3;
        c.small_src = start;
        c.small_dst = c.delta;
        c.small_n = a;
        c.ok = c.bulk_words <= ld;
    }
    return c;
}

// For a tile of a level-pair program: for every op term, whether it reads a
// window as loaded (its slot < load_cnt and not yet overwritten by an op of
// an earlier step; slots written in a step are read no earlier than the next
// step), and for every store whether its slot still holds a window (a copy
// tile).  TMA windows sit at a per-window word offset (alignment residue):
// exactly these reads must add it.
struct WindowReads {
    std::vector<std::array<int, 4>> term_window;  // per op of the tile: window index or -1
    std::vector<int> store_window;                // per store of the tile: window index or -1
};
WindowReads window_reads(const fhtb::FusedPass& ps, const fhtb::PassTile& t) {
    WindowReads w;
    std::vector<int> holds(static_cast<size_t>(std::max(ps.pmax_slots, t.load_cnt) + 1), -1);
    for (int k = 0; k < t.load_cnt; ++k) holds[static_cast<size_t>(k)] = k;
    for (int st = 0; st < t.nsteps; ++st) {
        const int ob = ps.pstep_offs[static_cast<size_t>(t.step_beg + st)];
        const int oe = ps.pstep_offs[static_cast<size_t>(t.step_beg + st + 1)];
        for (int oi = ob; oi < oe; ++oi) {
            const auto& op = ps.pops[static_cast<size_t>(oi)];
            std::array<int, 4> tw = {-1, -1, -1, -1};
            for (int k = 0; k < op.nterms; ++k) {
                const size_t sl = static_cast<size_t>(op.term[k].slot);
                tw[static_cast<size_t>(k)] = sl < holds.size() ? holds[sl] : -1;
            }
            w.term_window.push_back(tw);
        }
        for (int oi = ob; oi < oe; ++oi) {  // this step's outputs replace what their slots held
            const auto& op = ps.pops[static_cast<size_t>(oi)];
            for (int d : {op.dst, op.dst_hi})
                if (d >= 0) {
                    if (static_cast<size_t>(d) >= holds.size()) holds.resize(static_cast<size_t>(d) + 1, -1);
                    holds[static_cast<size_t>(d)] = -1;
                }
        }
    }
    for (int k = 0; k < t.store_cnt; ++k) {
        const auto& st = ps.pstores[static_cast<size_t>(t.store_beg + k)];
        const size_t sl = static_cast<size_t>(st.slot);
        w.store_window.push_back(sl < holds.size() ? holds[sl] : -1);
    }
    return w;
}

void upload(Group& g) {
    const SubPlan& sp = g.sp;
    // Width-32 non-root blocks go to the specialised K1P kernel (4-byte
    // accumulators); every other block to the table-driven K1.
    std::vector<int4> blocks;
    std::vector<int> by_x0;
    for (const auto& b : sp.blocks) {
        const bool by = g.use_by32 && !sp.root_is_block && sp.shapes[static_cast<size_t>(b.shape)].width == 32;
        if (by)
            by_x0.push_back(b.x0);
        else
            blocks.push_back(make_int4(b.x0, b.shape, b.depth, 0));
    }
    g.nblocks = static_cast<int>(blocks.size());
    g.nby = static_cast<int>(by_x0.size());
    std::vector<ShapeHdr> shapes;
    std::vector<int> step_offs;
    std::vector<fhtb::PassOp> k1_ops;
    const int mw = sp.max_block_width;
    for (const auto& s : sp.shapes) {
        ShapeHdr hdr{};
        hdr.width = s.width;
        hdr.nsteps = s.depth;
        hdr.op_base = static_cast<int>(k1_ops.size());
        hdr.step_base = static_cast<int>(step_offs.size());
        hdr.halo = s.halo;
        shapes.push_back(hdr);
        for (int o : s.step_offset) step_offs.push_back(o);
        // Step k (deepest first) reads buffer (nsteps-k)%2 and writes
        // (nsteps-1-k)%2; buffer p is slots [p*mw, (p+1)*mw) of the K1 tile.
        for (int k = 0; k < s.depth; ++k) {
            const int ps = ((s.depth - k) & 1) * mw, pd = ((s.depth - 1 - k) & 1) * mw;
            for (int o = s.step_offset[static_cast<size_t>(k)]; o < s.step_offset[static_cast<size_t>(k) + 1]; ++o) {
                const auto& op = s.ops[static_cast<size_t>(o)];
                fhtb::PassOp po{};
                po.dst = op.dst + pd;
                po.a = op.a + ps;
                po.b = op.b >= 0 ? op.b + ps : -1;
                po.ad = 0;
                po.bd = op.r;
                po.ext = s.extra[static_cast<size_t>(o)];
                k1_ops.push_back(po);
            }
        }
        g.dt.max_ops = std::max(g.dt.max_ops, static_cast<int>(s.ops.size()));
        g.dt.max_steps = std::max(g.dt.max_steps, s.depth);
    }
    // Assemble one blob, 16-byte aligned sections.
    std::vector<char> blob;
    auto put = [&](const void* p, size_t n) {
        size_t off = (blob.size() + 15) / 16 * 16;
        blob.resize(off + n);
        if (n) std::memcpy(blob.data() + off, p, n);
        return off;
    };
    const size_t o_blocks = put(blocks.data(), blocks.size() * sizeof(int4));
    const size_t o_by = put(by_x0.data(), by_x0.size() * sizeof(int));
    const size_t o_shapes = put(shapes.data(), shapes.size() * sizeof(ShapeHdr));
    const size_t o_steps = put(step_offs.data(), step_offs.size() * sizeof(int));
    const size_t o_k1 = put(k1_ops.data(), k1_ops.size() * sizeof(fhtb::PassOp));
    // the same ops baked into shared byte offsets (slot stride sr) for the
    // 4-byte vector executor: {dst, a, b aligned | (shift & 3) or -1, rows}
    std::vector<int4> k1_bops;
    {
        size_t k = 0;
        for (const auto& sh : sp.shapes)
            for (size_t o = 0; o < sh.ops.size(); ++o, ++k) {
                const fhtb::PassOp& po = k1_ops[k];
                const int64_t d = int64_t(po.dst) * g.sr * 4, a = int64_t(po.a) * g.sr * 4;
                const int64_t b = po.b < 0 ? -1 : ((int64_t(po.b) * g.sr + (po.bd & ~3)) * 4) | (po.bd & 3);
                k1_bops.push_back(make_int4(static_cast<int>(d), static_cast<int>(a), static_cast<int>(b), g.S + po.ext));
            }
    }
    const size_t o_k1b = put(k1_bops.data(), k1_bops.size() * sizeof(int4));
    struct PassOff {
        size_t tiles, loads, steps, ops, stores, bops, bops1 = 0, stores1 = 0;
        int pipe_delta = 0, pipe_loads = 0;
        size_t twin = 0, tbops = 0, tbops1 = 0;  // TMA window records and their ops (0: none)
        bool tma = false;
        size_t kwslots = 0, kwstores = 0;  // TMA windows in k2_pass (level pairs)
        bool ktma = false;
    };
    std::vector<PassOff> o_passes;
    for (const auto& ps : sp.passes) {
        static_assert(sizeof(fhtb::PassTile) == sizeof(fhtb::PassTileDev), "tile layout");
        static_assert(sizeof(fhtb::PassOp) == sizeof(fhtb::PassOpDev), "op layout");
        const PassProgram pr = program(ps, g.pairs);
        PassOff o{};
        o.tiles = put(pr.tiles.data(), pr.tiles.size() * sizeof(fhtb::PassTile));
        std::vector<int4> loads;
        for (const auto& l : ps.loads) loads.push_back(make_int4(l.gcol, l.slot, l.off, l.ext));
        o.loads = put(loads.data(), loads.size() * sizeof(int4));
        o.steps = put(pr.step_offs.data(), pr.step_offs.size() * sizeof(int));
        o.ops = put(ps.ops.data(), ps.ops.size() * sizeof(fhtb::PassOp));
        std::vector<int2> stores;
        for (const auto& st : pr.stores) {  // u16 pair mode: the root's upper-row slot in bits 16..
            if (st.slot >= (1 << 16) || st.slot_hi >= (1 << 15)) throw FhtError(FHT_ERR_INTERNAL, "slot index overflow");
            stores.push_back(make_int2(st.slot | (st.slot_hi >= 0 ? st.slot_hi << 16 : 0), st.gcol));
        }
        o.stores = put(stores.data(), stores.size() * sizeof(int2));
        // ops baked into shared byte offsets for the 4-byte kernel path
        {
            const int64_t L = g.pass_L[o_passes.size()], S = g.pass_S[o_passes.size()];
            std::vector<int4> bops;
            if (g.pairs) {  // 2 records per op: {dst, rows, nterms | (gcol+1) << 3, term0}, {term1, term2, term3, split}
                // ops of a tile's last step that produce a stored column carry
                // its global column: non-root bands store them from registers
                std::vector<int> gcol_of(ps.pops.size(), -1);
                for (const auto& t : ps.ptiles) {
                    if (t.nsteps == 0) continue;
                    const int lo = ps.pstep_offs[static_cast<size_t>(t.step_beg + t.nsteps - 1)];
                    const int hi = ps.pstep_offs[static_cast<size_t>(t.step_beg + t.nsteps)];
                    for (int o = lo; o < hi; ++o)
                        for (int k = 0; k < t.store_cnt; ++k) {
                            const auto& st = ps.pstores[static_cast<size_t>(t.store_beg + k)];
                            if (st.slot == ps.pops[static_cast<size_t>(o)].dst) gcol_of[static_cast<size_t>(o)] = st.gcol;
                        }
                }
                for (size_t oi = 0; oi < ps.pops.size(); ++oi) {
                    const auto& op = ps.pops[oi];
                    int64_t t[4] = {0, 0, 0, 0};
                    const int64_t esz = static_cast<int64_t>(g.acc_sz);
                    for (int k = 0; k < op.nterms; ++k) t[k] = (op.term[k].slot * L + op.term[k].off) * esz;
                    const int64_t d = op.dst * L * esz;
                    if (d > INT32_MAX || *std::max_element(t, t + 4) > INT32_MAX)
                        throw FhtError(FHT_ERR_INTERNAL, "op offset overflow");
                    if (gcol_of[oi] >= (1 << 27)) throw FhtError(FHT_ERR_INTERNAL, "column index overflow");
                    bops.push_back(make_int4(static_cast<int>(d), static_cast<int>(S + op.ext),
                                             op.nterms | ((gcol_of[oi] + 1) << 3), static_cast<int>(t[0])));
                    // u16 pair mode root ops: the upper-row slot's byte offset above the split
                    const int64_t dh = op.dst_hi >= 0 ? op.dst_hi * L * 4 : 0;
                    if (dh >= (int64_t(1) << 27)) throw FhtError(FHT_ERR_INTERNAL, "op offset overflow");
                    bops.push_back(make_int4(static_cast<int>(t[1]), static_cast<int>(t[2]), static_cast<int>(t[3]),
                                             op.split | static_cast<int>(dh << 4)));
                }
            }
            for (const auto& op : ps.ops) {
                if (g.pairs) break;
                const int64_t d = op.dst * L * 4, a = (op.a * L + op.ad) * 4;
                const int64_t b = op.b < 0 ? -1 : ((op.b * L + (op.bd & ~3)) * 4) | (op.bd & 3);
                if (d > INT32_MAX || a > INT32_MAX || b > INT32_MAX) throw FhtError(FHT_ERR_INTERNAL, "op offset overflow");
                bops.push_back(make_int4(static_cast<int>(d), static_cast<int>(a), static_cast<int>(b),
                                         static_cast<int>(S + op.ext)));
            }
            o.bops = put(bops.data(), bops.size() * sizeof(int4));
            // TMA windows for the level-pair k2_pass (row tiles: the windows'
            // starts, so their alignment residues, depend on the row tile and
            // are applied at run time): per op, the window index each term
            // reads (4 x u8, 0xff: an intermediate column); per store, bit 30
            // of the column marks a stored window (a copy tile)
            // (opt-in, FHT_K2_TMA_BANDS=1: measured slower -- these CTAs load one
            // row tile and then compute, so the bulk copies' latency is exposed;
            // c5 bands 0.684 / 0.900 -> 0.712 / 0.967 ms)
            if (g.pairs && esize_acc4(g) && env_int("FHT_K2_TMA_BANDS", 0, 0, 1) == 1) {
                bool ok = true;
                std::vector<int> wslots(ps.pops.size(), -1);
                std::vector<int2> wstores;
                for (const auto& st : pr.stores) wstores.push_back(make_int2(st.slot, st.gcol));
                for (const auto& t : ps.ptiles) {
                    if (t.load_cnt > 64) ok = false;  // residues of <= 64 windows live in two 64-bit masks
                    for (int k = 0; k < t.load_cnt; ++k) {
                        const auto& l = ps.loads[static_cast<size_t>(t.load_beg + k)];
                        if (l.slot != k || S + l.ext > g.sp.H) ok = false;
                    }
                    const WindowReads wr = window_reads(ps, t);
                    const int ob = ps.pstep_offs[static_cast<size_t>(t.step_beg)];
                    for (size_t i = 0; i < wr.term_window.size(); ++i) {
                        unsigned v = 0;
                        for (int k = 0; k < 4; ++k) {
                            const int win = wr.term_window[i][static_cast<size_t>(k)];
                            v |= static_cast<unsigned>(win < 0 ? 0xff : win) << (8 * k);
                        }
                        wslots[static_cast<size_t>(ob) + i] = static_cast<int>(v);
                    }
                    for (int k = 0; k < t.store_cnt; ++k)
                        if (wr.store_window[static_cast<size_t>(k)] >= 0)
                            wstores[static_cast<size_t>(t.store_beg + k)].y |= 1 << 30;
                }
                if (ok) {
                    o.kwslots = put(wslots.data(), wslots.size() * sizeof(int));
                    o.kwstores = put(wstores.data(), wstores.size() * sizeof(int2));
                    o.ktma = true;
                }
            }
            // u16 pair mode root band: the second-buffer variant for the
            // double-buffered kernel (load-space slots s < load_cnt -> s + delta)
            const bool last = o_passes.size() + 1 == sp.passes.size();
            if (g.pm_D && g.pairs && last && env_int("FHT_K2_PIPE", 1, 0, 1) == 1) {
                const int delta = ps.pmax_slots;
                int maxl = 0;
                for (const auto& t : ps.ptiles) maxl = std::max(maxl, t.load_cnt);
                std::vector<int4> b1 = bops;
                std::vector<int2> st1 = stores;
                auto mv = [&](int byteoff, int lc) {  // a baked byte offset slot*L*4 + off*4
                    const int64_t sl = byteoff / (L * 4);
                    return sl < lc ? static_cast<int>(byteoff + int64_t(delta) * L * 4) : byteoff;
                };
                for (const auto& t : ps.ptiles) {
                    const int lc = t.load_cnt;
                    const int ob = ps.pstep_offs[static_cast<size_t>(t.step_beg)];
                    const int oe = ps.pstep_offs[static_cast<size_t>(t.step_beg + t.nsteps)];
                    for (int oi = ob; oi < oe; ++oi) {
                        const auto& op = ps.pops[static_cast<size_t>(oi)];
                        int4& h = b1[2 * static_cast<size_t>(oi)];
                        int4& q = b1[2 * static_cast<size_t>(oi) + 1];
                        h.x = mv(h.x, lc);
                        if (op.nterms > 0) h.w = mv(h.w, lc);
                        if (op.nterms > 1) q.x = mv(q.x, lc);
                        if (op.nterms > 2) q.y = mv(q.y, lc);
                        if (op.nterms > 3) q.z = mv(q.z, lc);
                        if (op.dst_hi >= 0) q.w = op.split | (mv(static_cast<int>(op.dst_hi * L * 4), lc) << 4);
                    }
                    for (int k = 0; k < t.store_cnt; ++k) {
                        int2& r = st1[static_cast<size_t>(t.store_beg + k)];
                        int lo = r.x & 0xffff, hi = r.x >> 16;
                        if (lo < lc) lo += delta;
                        if (hi < lc) hi += delta;
                        if (lo >= (1 << 16) || hi >= (1 << 15)) throw FhtError(FHT_ERR_INTERNAL, "slot index overflow");
                        r.x = lo | (hi << 16);
                    }
                }
                const int64_t dh_max = int64_t(delta + maxl) * L * 4;
                if (dh_max >= (int64_t(1) << 27)) throw FhtError(FHT_ERR_INTERNAL, "op offset overflow");
                o.bops1 = put(b1.data(), b1.size() * sizeof(int4));
                o.stores1 = put(st1.data(), st1.size() * sizeof(int2));
                o.pipe_delta = delta;
                o.pipe_loads = maxl;
                // TMA windows (one row tile of all D words, s0 = 0): every
                // window's start is static, so the plan aligns it down to 16
                // bytes and folds the residue into the ops' term offsets.
                if (S >= g.pm_D && env_int("FHT_K2_TMA", 1, 0, 1) == 1) {
                    std::vector<int4> twin, tb = bops, tb1 = b1;
                    bool ok = true;
                    for (const auto& t : ps.ptiles) {
                        std::vector<int> delta_of(static_cast<size_t>(t.load_cnt), 0);
                        for (int k = 0; k < t.load_cnt; ++k) {
                            const auto& l = ps.loads[static_cast<size_t>(t.load_beg + k)];
                            const WinCopy c = window_copy(l.off, static_cast<int>(S + l.ext), g.sp.H, g.ld);
                            if (!c.ok) ok = false;
                            delta_of[static_cast<size_t>(k)] = c.delta;
                            const int dst = static_cast<int>(l.slot * L * 4);
                            twin.push_back(make_int4(l.gcol, dst + 4 * c.bulk_dst, c.bulk_src, c.bulk_words));
                            twin.push_back(make_int4(dst + 4 * c.small_dst, c.small_src, c.small_n, 0));
                            if (l.slot != k) ok = false;  // window k lives in slot k (load-space slots)
                        }
                        const int ob = ps.pstep_offs[static_cast<size_t>(t.step_beg)];
                        const int oe = ps.pstep_offs[static_cast<size_t>(t.step_beg + t.nsteps)];
                        const WindowReads wr = window_reads(ps, t);
                        for (int sw : wr.store_window)
                            if (sw >= 0) ok = false;  // a stored window (copy tile): not in the root band
                        for (int oi = ob; oi < oe; ++oi) {
                            const auto& op = ps.pops[static_cast<size_t>(oi)];
                            int4* rec[2] = {&tb[2 * static_cast<size_t>(oi)], &tb1[2 * static_cast<size_t>(oi)]};
                            for (int k = 0; k < op.nterms; ++k) {
                                const int win = wr.term_window[static_cast<size_t>(oi - ob)][static_cast<size_t>(k)];
                                if (win < 0) continue;  // an intermediate column
                                const int add = 4 * delta_of[static_cast<size_t>(win)];
                                for (int4* r : rec) {
                                    int& f = k == 0 ? r[0].w : k == 1 ? r[1].x : k == 2 ? r[1].y : r[1].z;
                                    f += add;
                                }
                            }
                        }
                    }
                    if (ok) {
                        o.twin = put(twin.data(), twin.size() * sizeof(int4));
                        o.tbops = put(tb.data(), tb.size() * sizeof(int4));
                        o.tbops1 = put(tb1.data(), tb1.size() * sizeof(int4));
                        o.tma = true;
                    }
                }
            }
        }
        o_passes.push_back(o);
    }
    blob.resize(blob.size() + 16);
    cuda_check(counted_malloc(&g.dt.blob, blob.size()), "counted_malloc(plan tables)");
    cuda_check(cudaMemcpy(g.dt.blob, blob.data(), blob.size(), cudaMemcpyHostToDevice), "cudaMemcpy(plan tables)");
    char* base = static_cast<char*>(g.dt.blob);
    g.dt.blocks = reinterpret_cast<const int4*>(base + o_blocks);
    g.dt.by_x0 = reinterpret_cast<const int*>(base + o_by);
    g.dt.shapes = reinterpret_cast<const ShapeHdr*>(base + o_shapes);
    g.dt.step_offs = reinterpret_cast<const int*>(base + o_steps);
    g.dt.k1_ops = reinterpret_cast<const fhtb::PassOpDev*>(base + o_k1);
    g.dt.k1_bops = reinterpret_cast<const int4*>(base + o_k1b);
    for (size_t i = 0; i < o_passes.size(); ++i) {
        const PassOff& o = o_passes[i];
        fhtb::PassDev d{};
        d.tiles = reinterpret_cast<const fhtb::PassTileDev*>(base + o.tiles);
        d.loads = reinterpret_cast<const int4*>(base + o.loads);
        d.step_offs = reinterpret_cast<const int*>(base + o.steps);
        d.ops = reinterpret_cast<const fhtb::PassOpDev*>(base + o.ops);
        d.stores = reinterpret_cast<const int2*>(base + o.stores);
        d.bops = reinterpret_cast<const int4*>(base + o.bops);
        d.bops1 = o.pipe_delta ? reinterpret_cast<const int4*>(base + o.bops1) : nullptr;
        d.stores1 = o.pipe_delta ? reinterpret_cast<const int2*>(base + o.stores1) : nullptr;
        d.pipe_delta = o.pipe_delta;
        d.pipe_loads = o.pipe_loads;
        d.tma = o.tma ? 1 : 0;
        d.twin = o.tma ? reinterpret_cast<const int4*>(base + o.twin) : nullptr;
        d.tbops = o.tma ? reinterpret_cast<const int4*>(base + o.tbops) : nullptr;
        d.tbops1 = o.tma ? reinterpret_cast<const int4*>(base + o.tbops1) : nullptr;
        d.ktma = o.ktma ? 1 : 0;
        d.kwslots = o.ktma ? reinterpret_cast<const int*>(base + o.kwslots) : nullptr;
        d.kwstores = o.ktma ? reinterpret_cast<const int2*>(base + o.kwstores) : nullptr;
        d.tile_nc_max = 0;
        for (const auto& t : program(sp.passes[i], g.pairs).tiles) d.tile_nc_max = std::max(d.tile_nc_max, t.store_cnt);
        d.S = g.pass_S[i];
        d.L = g.pass_L[i];
        const PassProgram pr = program(sp.passes[i], g.pairs);
        d.ntiles = static_cast<int>(pr.tiles.size());
        d.max_slots = pr.max_slots;
        d.max_tile_ops = pr.max_tile_ops();
        d.pairs = g.pairs ? 1 : 0;
        g.dt.passes.push_back(d);
    }
}


// Rows per K2 row tile for a pass: as many as fit `budget` bytes of shared
// memory (max_slots slots of S + max_ext rows), capped at H; multiples of 32.
int pass_rows(const fhtb::FusedPass& ps, int max_slots, int H, size_t esz, size_t budget) {
    const long cap = static_cast<long>(budget / (esz * static_cast<size_t>(std::max(1, max_slots)))) - ps.max_ext - 20;
    if (cap >= H) return H;
    if (cap < 32) return static_cast<int>(std::max(0L, cap));
    return static_cast<int>(cap / 32 * 32);
}

int block_width_default() { return env_int("FHT_BLOCK_WIDTH", 32, 1, 64); }

// k1_acc32: an int64 plan whose pass 0 may accumulate in int32 (the caller
// knows 32 * max|v| < 2^31; the int64 reference entry points, run_i64)
fht_plan_s* create_plan(int w, int h, int strategy, int in, int acc, int out, int mask, int batch, int layout,
                        int device, bool k1_acc32 = false) {
    if (w < 1 || h < 1) throw std::invalid_argument("fht2d: image is empty");
    if (strategy != FHT_SPLIT_SIMPLE && strategy != FHT_SPLIT_TWEAKED)
        throw std::invalid_argument("unknown strategy (expected simple|tweaked)");
    if (!valid_types(in, acc, out)) throw std::invalid_argument("unsupported (input, accumulator, output) dtype triple");
    if (mask < 1 || mask > 15) throw std::invalid_argument("quadrant mask must select 1..4 quadrants");
    if (batch < 1) throw std::invalid_argument("batch must be >= 1");
    if (layout != FHT_LAYOUT_REFERENCE && layout != FHT_LAYOUT_NATIVE) throw std::invalid_argument("unknown layout");
    if (static_cast<int64_t>(w) * h > (int64_t(1) << 31) - 1) throw std::invalid_argument("image too large");
    // Static overflow budget for u8 into int32 (transform.cpp:16-27 with vmax = 255).
    const bool uses_h = (mask & (FHT_VERT_POS | FHT_VERT_NEG)) != 0, uses_w = (mask & 3) != 0;
    const int64_t wmax = std::max<int64_t>(uses_w ? w : 0, uses_h ? h : 0);
    if (in == FHT_U8 && acc == FHT_I32 && wmax * 255 >= (int64_t(1) << 31))
        throw std::overflow_error("fht2d: width * 255 reaches 2^31; use an int64 accumulator");
    int ndev = 0;
    cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw std::invalid_argument("no such CUDA device");
    DeviceGuard dg(device);

    auto p = std::make_unique<fht_plan_s>();
    cuda_check(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
    cuda_check(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming), "cudaEventCreate");
    p->w = w, p->h = h, p->strategy = strategy, p->in = in, p->acc = acc, p->out = out, p->mask = mask;
    p->batch = batch, p->layout = layout, p->device = device;
    const int bw = block_width_default();
    const size_t acc_sz = esize(acc);

    // Orientation groups: horizontal quadrants work on (W=w, H=h), vertical on
    // (W=h, H=w).  A square image shares one table set across all four.
    std::vector<std::pair<int, std::vector<int>>> orient;  // (horizontal?, codes)
    std::vector<int> hq, vq;
    for (int q = 0; q < 4; ++q)
        if (mask & (1 << q)) (q < 2 ? hq : vq).push_back(q);
    if (w == h) {
        std::vector<int> all = hq;
        all.insert(all.end(), vq.begin(), vq.end());
        orient.push_back({1, all});
    } else {
        if (!hq.empty()) orient.push_back({1, hq});
        if (!vq.empty()) orient.push_back({0, vq});
    }
    size_t max_slot_bytes = 0;
    int max_nq = 0;
    for (auto& [horizontal, codes] : orient) {
        auto g = std::make_unique<Group>();
        const int W = horizontal ? w : h, H = horizontal ? h : w;
        // Fused-pass tiles: shrink the tile width until every pass gets a
        // reasonable row tile in the shared-memory budget.
        const size_t budget = static_cast<size_t>(env_int("FHT_K2_SMEM_KB", 105, 16, 220)) * 1024;
        const int levels = env_int("FHT_PASS_LEVELS", 5, 1, 8);
        int tw = env_int("FHT_TILE_WIDTH", 32, 1, 64);  // K2's root store handles <= 64 slopes per tile
        g->pairs = (acc_sz == 4 || acc_sz == 8) && env_int("FHT_K2_PAIRS", 1, 0, 1) == 1;
        // u16 pair mode: u8 images whose root children are at
        // most 257 wide (every non-root node sum < 2^16) and H <= 512 (one
        // K1P/K2 row tile of D = H/2 rounded up to 8 words).  It needs the
        // staged K1P (variant 5) and a single K2 band; FHT_U16_PAIRS=0 turns it off.
        const int pmD = round_up((H + 1) / 2, 8);
        bool pm = false;
        {
            const auto wc = fhtb::split_width(std::max(W, 2), strategy);
            const int stage_env0 = env_int("FHT_K1_STAGE", -1, -1, 1);
            pm = in == FHT_U8 && acc == FHT_I32 && g->pairs && env_int("FHT_U16_PAIRS", 1, 0, 1) == 1 &&
                 env_int("FHT_K1_BY32", 1, 0, 1) == 1 && env_int("FHT_K1P_VARIANT", 5, 0, 5) == 5 && stage_env0 != 0 &&
                 bw == 32 && W > 2 * bw && H >= 64 && pmD <= 256 && pmD <= H && std::max(wc.first, wc.second) <= 257;
        }
        // pair mode: 16-slope tiles (the root's upper-row slots then leave room
        // for one row tile of all D words at two CTAs per SM; measured faster)
        if (pm && !std::getenv("FHT_TILE_WIDTH")) tw = 16;
        for (;;) {
            g->sp = SubPlan::build(W, H, strategy, bw, levels, tw, pm);
            bool ok = true;
            for (const auto& ps : g->sp.passes) {
                const PassProgram pr = program(ps, g->pairs);
                const int rows = pass_rows(ps, pr.max_slots, H, acc_sz, budget);
                const int Lmax = std::min(rows, env_int("FHT_K2_SMAX", 256, 32, 4096)) + ps.max_ext + 20;
                ok = ok && rows >= std::min(H, 32) &&
                     fhtb::k2_smem_bytes(acc, pr.max_slots, Lmax, pr.max_tile_ops()) <= 227 * 1024;
            }
            if (pm) {  // one K2 band, row tiles of >= 64 words (or all D)
                const auto& ps = g->sp.passes;
                const bool fit = ps.size() == 1 && pass_rows(ps[0], program(ps[0], g->pairs).max_slots, H, acc_sz,
                                                             budget) >= std::min(pmD, 64);
                if (!fit) {
                    pm = false;
                    tw = env_int("FHT_TILE_WIDTH", 32, 1, 64);
                    continue;  // rebuild without the root's upper-row slots
                }
            }
            if (ok) break;
            if (tw == 1) throw FhtError(FHT_ERR_INTERNAL, "fused pass does not fit shared memory");
            tw = std::max(1, tw / 2);
        }
        g->pm_D = pm ? pmD : 0;
        // int64 accumulation with pass 0 in int32: blocks of width <= 32
        // (Simple trees with a wider root block keep int64 pass 0)
        g->k1_acc32 = k1_acc32 && acc_sz == 8 && in != FHT_U8 && in != FHT_F32 && bw <= 32 &&
                      env_int("FHT_K1_ACC32", 1, 0, 1) == 1;
        g->acc_sz = acc_sz;
        g->qs.n = static_cast<int>(codes.size());
        for (int k = 0; k < 4; ++k) g->qs.code[k] = k < g->qs.n ? codes[static_cast<size_t>(k)] : 0;
        g->ld = round_up(H, acc_sz == 8 ? 16 : 32);
        // K1 rows per tile: every op's window (S + halo) fits the executor's
        // 256-row item pair.
        // K1 rows per tile: the fewest tiles of <= 256 rows, balanced.
        const int smax = acc_sz == 8 && !g->k1_acc32 ? 128 : env_int("FHT_K1_SMAX", 256, 16, 256);
        const int ntile = (H + smax - 1) / smax;
        int S = ((H + ntile - 1) / ntile + 7) & ~7;
        if (H < S) S = H;
        if (pm) S = pmD;  // one tile of D words (rows [0, 2D))
        g->S = S;
        // K1 column stride: 16-byte aligned, vector-merge slack, and room for
        // the row-major staging tile of the horizontal loader (R x (wb+1)).
        {
            const int R = S + g->sp.max_halo, mw = std::max(1, g->sp.max_block_width);
            int sr = std::max(R + 12, (R * (mw + 1) + mw - 1) / mw);
            sr = (sr + 3) & ~3;
            if (((sr >> 2) & 1) == 0) sr += 4;
            g->sr = sr;
        }
        g->nbuf = g->sp.root_is_block ? 0 : (g->sp.passes.size() > 1 ? 2 : 1);
        g->use_by32 = (acc_sz == 4 || g->k1_acc32) && env_int("FHT_K1_BY32", 1, 0, 1) == 1;
        // staging pays off once the batch is large (its launch costs a few
        // microseconds: a loss for one small image); FHT_K1_STAGE=0/1 forces it
        const int stage_env = env_int("FHT_K1_STAGE", -1, -1, 1);
        const bool stage_on =
            pm || (stage_env < 0 ? static_cast<int64_t>(batch) * w * h >= (int64_t(8) << 20) : stage_env == 1);
        if (in == FHT_U8 && g->use_by32 && stage_on) {
            // columns of ntile * S + 31 rows (+ the last 4-byte word), 16-byte aligned
            bool need_t = false, need_p = false;
            for (int k = 0; k < g->qs.n; ++k) (codes[static_cast<size_t>(k)] < 2 ? need_t : need_p) = true;
            const long long ntile = (H + S - 1) / S;
            // pair mode: rows [0, 2D + 31) (the upper half of every word is D rows on)
            // FHT_STAGE_ALIGN=128 starts every column on a 128-byte line (a warp's
            // 4-byte loads of 32 row chunks then touch one line, not two):
            // measured slower (the staging writes grow 14 %, K1P unchanged)
            const long long al = env_int("FHT_STAGE_ALIGN", 16, 16, 128);
            g->stage_pitch = ((pm ? 2LL * pmD : ntile * S) + 36 + al - 1) / al * al;
            const long long set = static_cast<long long>(W) * g->stage_pitch;
            g->stage_t = need_t ? 0 : -1;
            g->stage_p = need_p ? (need_t ? set : 0) : -1;
            g->stage_img = set * ((need_t ? 1 : 0) + (need_p ? 1 : 0));
        }
        g->slot_bytes = static_cast<size_t>(g->nbuf) * W * g->ld * acc_sz;
        for (size_t i = 0; i < g->sp.passes.size(); ++i) {
            int S2 = std::min(env_int("FHT_K2_SMAX", 256, 32, 4096),
                              pass_rows(g->sp.passes[i], program(g->sp.passes[i], g->pairs).max_slots, H, acc_sz, budget));
            if (!pm) {  // balance the row tiles
                const int nt = (H + S2 - 1) / std::max(1, S2);
                S2 = std::min(S2, ((H + nt - 1) / nt + 7) & ~7);
                if (S2 > H) S2 = H;
            }
            if (pm) {  // row tiles over the D words, balanced
                S2 = std::min(S2, pmD);
                const int nt = (pmD + S2 - 1) / S2;
                S2 = ((pmD + nt - 1) / nt + 7) & ~7;
            }
            // slot capacity: window + vector-merge slack, a multiple of 4 rows
            // (16-byte aligned slots) with L/4 odd (spreads the transposed
            // root stores over the banks)
            int L2 = (S2 + g->sp.passes[i].max_ext + 12 + 3) & ~3;
            if (((L2 >> 2) & 1) == 0) L2 += 4;
            g->pass_S.push_back(S2);
            g->pass_L.push_back(L2);
        }
        upload(*g);
        // grid.y carries blocks / tiles: 65535 of them at most
        bool fits = g->nby <= 65535 && g->nblocks <= 65535;
        for (const auto& d : g->dt.passes) fits = fits && d.ntiles <= 65535;
        if (!fits) throw std::invalid_argument("fht2d: working width too large (more than 65535 tiles per pass)");
        const size_t smem = fhtb::k1_smem_bytes(g->k1_acc32 ? FHT_I32 : acc, g->sp.max_block_width, g->sr, g->dt.max_ops,
                                                g->dt.max_steps);
        if (smem > 227 * 1024) throw FhtError(FHT_ERR_INTERNAL, "K1 tile exceeds shared memory");
        max_slot_bytes = std::max(max_slot_bytes, g->slot_bytes * g->qs.n);
        if (g->nby > 0 || g->pm_D) p->stage_bytes_img = std::max(p->stage_bytes_img, static_cast<size_t>(g->stage_img));
        max_nq = std::max(max_nq, g->qs.n);
        p->additions += g->sp.additions * static_cast<uint64_t>(g->qs.n) * static_cast<uint64_t>(batch);
        p->groups.push_back(std::move(g));
    }
    // Images per chunk: all of them unless FHT_CHUNK_IMAGES asks otherwise or
    // grid.z (65535 slots) / the 16 GiB workspace cap forces a split.
    int chunk = batch;
    if (const char* e = std::getenv("FHT_CHUNK_IMAGES")) chunk = std::max(1, std::min(batch, std::atoi(e)));
    chunk = std::min(chunk, 65535 / std::max(1, max_nq));
    const size_t cap = size_t(16) << 30;
    const size_t per_img = max_slot_bytes + p->stage_bytes_img;
    if (per_img > 0) chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(chunk, cap / per_img)));
    p->chunk = chunk;
    p->slot_bytes_img = max_slot_bytes;
    p->ws_bytes = per_img * static_cast<size_t>(chunk);
    const int nchunks = (batch + chunk - 1) / chunk;
    int per_chunk = 0;
    for (auto& g : p->groups)
        per_chunk += (g->nblocks > 0 ? 1 : 0) + (g->nby > 0 ? 1 : 0) + ((g->nby > 0 || g->pm_D) && g->stage_img > 0 ? 1 : 0) +
                     static_cast<int>(g->sp.passes.size());
    p->launches = per_chunk * nchunks;
    return p.release();
}

struct PeerOut {  // fht_execute_pitched_peer: slopes [c0, c1) also stored to `ptr`
    void* ptr = nullptr;
    int c0 = 0, c1 = 0;
};

void execute(fht_plan_s* p, const void* d_in, int64_t in_stride, void* const d_out[4], int64_t out_stride,
             void* ws, cudaStream_t st, fhtb::LaunchHook hook = nullptr, void* ctx = nullptr, int64_t in_pitch = 0,
             int img_begin = 0, int img_end = -1, PeerOut peer = {}) {
    if (img_end < 0) img_end = p->batch;
    if (in_pitch == 0) in_pitch = p->w;
    if (in_pitch < p->w) throw std::invalid_argument("fht_execute: row pitch smaller than the image width");
    if (!d_in) throw std::invalid_argument("fht_execute: null input");
    for (int q = 0; q < 4; ++q)
        if ((p->mask & (1 << q)) && !d_out[q]) throw std::invalid_argument("fht_execute: null output for a selected quadrant");
    if (p->ws_bytes && !ws) throw std::invalid_argument("fht_execute: null workspace");
    DeviceGuard dg(p->device);
    nvtxRangePushA("fht_execute");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    for (int img0 = img_begin; img0 < img_end; img0 += p->chunk) {
        const int nimg = std::min(p->chunk, img_end - img0);
        for (auto& gp : p->groups) {
            Group& g = *gp;
            GroupLaunch L{};
            L.img = d_in;
            L.in_dtype = p->in;
            L.img_w = p->w;
            L.img_h = p->h;
            L.img_pitch = in_pitch;
            L.img_stride = in_stride;
            L.img0 = img0;
            L.nimg = nimg;
            L.qs = g.qs;
            L.W = g.sp.W;
            L.H = g.sp.H;
            L.ld = g.ld;
            L.acc_dtype = p->acc;
            L.S = g.S;
            L.nblocks = g.nblocks;
            L.blocks = g.dt.blocks;
            L.nby = g.nby;
            L.by_x0 = g.dt.by_x0;
            L.k1p_variant = g.pm_D ? 5 : env_int("FHT_K1P_VARIANT", 5, 0, 5);  // see GroupLaunch
            L.k1_acc32 = g.k1_acc32 ? 1 : 0;
            L.pm_D = g.pm_D;
            L.k1p_pair576 = env_int("FHT_K1P_PAIR576", 1, 0, 1);
            L.k1p_576 = env_int("FHT_K1P_576", 1, 0, 1);
            L.k2_scalar = env_int("FHT_K2_SCALAR", 1, 0, 1);
            L.k2_bulk = env_int("FHT_K2_BULK", 0, 0, 1);
            L.pdl = env_int("FHT_PDL", 1, 0, 1);
            L.aux_stream = env_int("FHT_K1_OVERLAP", 1, 0, 1) ? p->aux : nullptr;
            L.ev_fork = p->ev_fork;
            L.ev_join = p->ev_join;
            L.fork_mu = &p->fork_mu;
            L.shapes = g.dt.shapes;
            L.step_offs = g.dt.step_offs;
            L.k1_ops = g.dt.k1_ops;
            L.k1_bops = g.dt.k1_bops;
            L.k1_max_ops = g.dt.max_ops;
            L.k1_max_steps = g.dt.max_steps;
            L.k1_max_width = g.sp.max_block_width;
            L.k1_sr = g.sr;
            L.root_is_block = g.sp.root_is_block;
            L.npasses = static_cast<int>(g.dt.passes.size());
            L.passes = g.dt.passes.data();
            L.ws = ws;
            L.nbuf = g.nbuf;
            // staging after this chunk's slot buffers (execute_host parts hand
            // each call a workspace sized for its own images)
            L.stage = g.stage_img > 0 ? static_cast<unsigned char*>(ws) + p->slot_bytes_img * static_cast<size_t>(nimg)
                                      : nullptr;
            L.stage_pitch = g.stage_pitch;
            L.stage_img = g.stage_img;
            L.stage_t = g.stage_t;
            L.stage_p = g.stage_p;
            for (int q = 0; q < 4; ++q) L.out.ptr[q] = d_out[q];
            L.out.img_stride = out_stride;
            L.out.layout = p->layout;
            L.out.dtype = p->out;
            L.out.peer = peer.ptr;
            L.out.peer_c0 = peer.c0;
            L.out.peer_c1 = peer.c1;
            if (fhtb::launch_group(L, st, hook, ctx) < 0) throw FhtError(FHT_ERR_INVALID, "unsupported dtype triple");
            cuda_check(cudaGetLastError(), "kernel launch");
        }
    }
}

size_t cells_of(const fht_plan_s* p) { return static_cast<size_t>(p->w) * p->h; }

// Host buffers in and out.  For batches the images are cut into parts that
// rotate over three plan-owned streams, so the H2D copy of one part, the
// kernels of another and the D2H copies of a third overlap (PCIe is full
// duplex; the transform itself is a few percent of the copy time).
void execute_host(fht_plan_s* p, const void* h_in, void* const h_out[4], cudaStream_t st) {
    if (!h_in) throw std::invalid_argument("fht_execute_host: null input");
    for (int q = 0; q < 4; ++q)
        if ((p->mask & (1 << q)) && !h_out[q]) throw std::invalid_argument("fht_execute_host: null output for a selected quadrant");
    std::lock_guard<std::mutex> lk(p->host_mu);
    DeviceGuard dg(p->device);
    const size_t cells = cells_of(p);
    const size_t in_img = cells * esize(p->in), out_img = cells * esize(p->out);
    const int nparts = p->batch >= 2 ? std::min(p->batch, env_int("FHT_HOST_PARTS", 8, 1, 64)) : 1;
    const int nst = nparts > 1 ? kHostStreams : 1;
    const int per_part = (p->batch + nparts - 1) / nparts;
    const size_t ws_per_img = p->chunk ? p->ws_bytes / static_cast<size_t>(p->chunk) : 0;
    const size_t ws_part = ws_per_img * static_cast<size_t>(std::min(per_part, p->chunk));
    if (!p->st_in) cuda_check(counted_malloc(&p->st_in, in_img * p->batch), "counted_malloc(staging in)");
    for (int q = 0; q < 4; ++q)
        if ((p->mask & (1 << q)) && !p->st_out[q])
            cuda_check(counted_malloc(&p->st_out[q], out_img * p->batch), "counted_malloc(staging out)");
    if (ws_part && !p->st_ws) cuda_check(counted_malloc(&p->st_ws, ws_part * nst), "counted_malloc(workspace)");
    if (nst > 1 && !p->hst[0]) {
        for (int k = 0; k < kHostStreams; ++k) {
            cuda_check(cudaStreamCreateWithFlags(&p->hst[k], cudaStreamNonBlocking), "cudaStreamCreate");
            cuda_check(cudaEventCreateWithFlags(&p->hev[k], cudaEventDisableTiming), "cudaEventCreate");
        }
        cuda_check(cudaEventCreateWithFlags(&p->hev_start, cudaEventDisableTiming), "cudaEventCreate");
    }
    if (nst > 1) {  // order after the caller's stream
        cuda_check(cudaEventRecord(p->hev_start, st), "cudaEventRecord");
        for (int k = 0; k < nst; ++k) cuda_check(cudaStreamWaitEvent(p->hst[k], p->hev_start, 0), "cudaStreamWaitEvent");
    }
    for (int part = 0; part < nparts; ++part) {
        const int b = part * per_part, e = std::min(p->batch, b + per_part);
        if (b >= e) break;
        cudaStream_t s = nst > 1 ? p->hst[part % nst] : st;
        char* ws = static_cast<char*>(p->st_ws) + (nst > 1 ? (part % nst) * ws_part : 0);
        cuda_check(cudaMemcpyAsync(static_cast<char*>(p->st_in) + b * in_img, static_cast<const char*>(h_in) + b * in_img,
                                   (e - b) * in_img, cudaMemcpyHostToDevice, s), "H2D");
        execute(p, p->st_in, static_cast<int64_t>(cells), p->st_out, static_cast<int64_t>(cells), ws, s, nullptr, nullptr,
                0, b, e);
        for (int q = 0; q < 4; ++q)
            if (p->mask & (1 << q))
                cuda_check(cudaMemcpyAsync(static_cast<char*>(h_out[q]) + b * out_img,
                                           static_cast<char*>(p->st_out[q]) + b * out_img, (e - b) * out_img,
                                           cudaMemcpyDeviceToHost, s), "D2H");
    }
    if (nst > 1) {
        for (int k = 0; k < nst; ++k) {
            cuda_check(cudaEventRecord(p->hev[k], p->hst[k]), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(st, p->hev[k], 0), "cudaStreamWaitEvent");
        }
    }
    cuda_check(counted_sync(st), "cudaStreamSynchronize");
}

// absmax on device -> (ok_for_i32, within 2^62 budget)
void check_budget(const void* d_in, int dtype, int64_t count, int width, int* ok_i32, cudaStream_t st,
                  unsigned long long* vmax_out = nullptr) {
    if (dtype == FHT_U8) {
        if (ok_i32) *ok_i32 = static_cast<int64_t>(width) * 255 < (int64_t(1) << 31);
        return;
    }
    if (dtype == FHT_F32) throw std::invalid_argument("check_budget: integer inputs only");
    unsigned long long* d_max = nullptr;
    cuda_check(counted_malloc_async(reinterpret_cast<void**>(&d_max), sizeof(unsigned long long), st), "cudaMallocAsync");
    cuda_check(cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), st), "cudaMemsetAsync");
    fhtb::launch_absmax(d_in, dtype, count, d_max, st);
    unsigned long long vmax = 0;
    cuda_check(cudaMemcpyAsync(&vmax, d_max, sizeof(vmax), cudaMemcpyDeviceToHost, st), "D2H(absmax)");
    cuda_check(cudaFreeAsync(d_max, st), "cudaFreeAsync");
    cuda_check(counted_sync(st), "cudaStreamSynchronize");
    const unsigned __int128 prod = static_cast<unsigned __int128>(static_cast<unsigned>(width)) * vmax;
    if (prod >= (static_cast<unsigned __int128>(1) << 62))
        throw std::overflow_error("fht2d: width * max|value| reaches 2^62; sums could overflow 64-bit accumulators");
    if (vmax_out) *vmax_out = vmax;
    if (ok_i32) *ok_i32 = prod < (static_cast<unsigned __int128>(1) << 31);
}

// Per-device cache of plans used by the int64 reference entry points:
// least-recently-used, at most FHT_PLAN_CACHE (default 8) plans, so a process
// that transforms many image sizes does not keep a stream, events and device
// tables for each forever.  Entries are shared_ptrs: a plan evicted while
// another thread executes it lives until that call returns.  The cache object
// is deliberately never destroyed (a static destructor would run after the
// CUDA runtime's teardown); fht_plan_cache_clear releases it explicitly.
using CacheKey = std::tuple<int, int, int, int, int, int>;
struct PlanCache {
    std::mutex mu;
    std::list<std::pair<CacheKey, std::shared_ptr<fht_plan_s>>> lru;  // front = most recent
};
PlanCache& plan_cache() {
    static PlanCache* c = new PlanCache;
    return *c;
}

std::shared_ptr<fht_plan_s> cached_plan(int w, int h, int strategy, int acc, int mask, int device,
                                        bool k1_acc32 = false) {
    PlanCache& c = plan_cache();
    const auto key = std::make_tuple(w, h, strategy, acc + (k1_acc32 ? 1000 : 0), mask, device);
    {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.lru.begin(); it != c.lru.end(); ++it)
            if (it->first == key) {
                c.lru.splice(c.lru.begin(), c.lru, it);
                return it->second;
            }
    }
    // build outside the lock (plan creation uploads tables); a racing thread
    // may build the same plan, the first insert wins
    std::shared_ptr<fht_plan_s> p(
        create_plan(w, h, strategy, FHT_I64, acc, FHT_I64, mask, 1, FHT_LAYOUT_REFERENCE, device, k1_acc32));
    std::vector<std::shared_ptr<fht_plan_s>> evicted;  // destroyed after the lock is released
    {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto& e : c.lru)
            if (e.first == key) return e.second;
        c.lru.emplace_front(key, p);
        const size_t cap = static_cast<size_t>(env_int("FHT_PLAN_CACHE", 8, 1, 1024));
        while (c.lru.size() > cap) {
            evicted.push_back(std::move(c.lru.back().second));
            c.lru.pop_back();
        }
    }
    return p;
}

// The root merge's slope table (t, t0, t1, r) per (W, H, strategy, device):
// built and uploaded once, then shared (immutable) by every call, so the
// multi-GPU root split's timed step neither allocates nor synchronises.  A
// few bytes per slope; kept for the life of the process.
const int4* merge_root_table(int width, int height, int strategy) {
    static std::mutex mu;
    static auto* tables = new std::map<std::tuple<int, int, int, int>, int4*>;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(width, height, strategy, dev);
    auto it = tables->find(key);
    if (it != tables->end()) return it->second;
    const auto [w0, w1] = fhtb::split_width(width, strategy);
    std::vector<int4> ops(static_cast<size_t>(width));
    for (int t = 0; t < width; ++t) {  // transform.cpp:46-49
        const int t0 = static_cast<int>(fhtb::round_half_up_ratio(static_cast<int64_t>(t) * (w0 - 1), width - 1));
        const int t1 = static_cast<int>(fhtb::round_half_up_ratio(static_cast<int64_t>(t) * (w1 - 1), width - 1));
        ops[static_cast<size_t>(t)] = make_int4(t, t0, t1, (t - t1) % height);
    }
    int4* d_ops = nullptr;
    cuda_check(counted_malloc(reinterpret_cast<void**>(&d_ops), ops.size() * sizeof(int4)), "counted_malloc(merge table)");
    cuda_check(cudaMemcpy(d_ops, ops.data(), ops.size() * sizeof(int4), cudaMemcpyHostToDevice), "H2D(merge table)");
    tables->emplace(key, d_ops);
    return d_ops;
}

size_t plan_cache_clear() {
    PlanCache& c = plan_cache();
    std::list<std::pair<CacheKey, std::shared_ptr<fht_plan_s>>> gone;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        gone.swap(c.lru);
    }
    return gone.size();
}

size_t plan_cache_size() {
    PlanCache& c = plan_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    return c.lru.size();
}

void run_i64(const int64_t* img, int w, int h, int strategy, int mask, int64_t* const outs[4], uint64_t* adds) {
    if (w < 1 || h < 1 || !img) throw std::invalid_argument("fht2d: image is empty");
    if (strategy != FHT_SPLIT_SIMPLE && strategy != FHT_SPLIT_TWEAKED)
        throw std::invalid_argument("unknown strategy (expected simple|tweaked)");
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cudaStream_t st = cudaStreamPerThread;
    const size_t cells = static_cast<size_t>(w) * h;
    void* d_in = nullptr;
    void* d_out[4] = {nullptr, nullptr, nullptr, nullptr};
    void* d_ws = nullptr;
    auto release = [&] {
        if (d_in) cudaFreeAsync(d_in, st);
        for (void* q : d_out)
            if (q) cudaFreeAsync(q, st);
        if (d_ws) cudaFreeAsync(d_ws, st);
        counted_sync(st);
    };
    try {
        cuda_check(counted_malloc_async(&d_in, cells * 8, st), "counted_malloc_async(in)");
        cuda_check(cudaMemcpyAsync(d_in, img, cells * 8, cudaMemcpyHostToDevice, st), "H2D");
        // check_overflow_budget (transform.cpp:16-27) for every quadrant's working width.
        int ok32 = 0;
        unsigned long long vmax = 0;
        const int wmax = std::max((mask & 3) ? w : 0, (mask & 12) ? h : 0);
        check_budget(d_in, FHT_I64, static_cast<int64_t>(cells), wmax, &ok32, st, &vmax);
        // int64 sums needed, but width-32 blocks stay inside int32: pass 0 in int32
        const bool k1_32 = !ok32 && 32ull * vmax < (1ull << 31);
        const std::shared_ptr<fht_plan_s> sp = cached_plan(w, h, strategy, ok32 ? FHT_I32 : FHT_I64, mask, dev, k1_32);
        fht_plan_s* p = sp.get();
        for (int q = 0; q < 4; ++q)
            if (mask & (1 << q)) cuda_check(counted_malloc_async(&d_out[q], cells * 8, st), "counted_malloc_async(out)");
        if (p->ws_bytes) cuda_check(counted_malloc_async(&d_ws, p->ws_bytes, st), "counted_malloc_async(ws)");
        execute(p, d_in, static_cast<int64_t>(cells), d_out, static_cast<int64_t>(cells), d_ws, st);
        for (int q = 0; q < 4; ++q)
            if (mask & (1 << q)) cuda_check(cudaMemcpyAsync(outs[q], d_out[q], cells * 8, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(counted_sync(st), "cudaStreamSynchronize");
        if (adds) *adds = p->additions;
    } catch (...) {
        release();
        throw;
    }
    release();
}

}  // namespace

extern "C" {

int fht_plan_create(int width, int height, int strategy, int in_dtype, int acc_dtype, int out_dtype,
                    int quadrant_mask, int batch, int layout, int device, fht_plan_t* plan) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan pointer");
        const bool p0 = acc_dtype == FHT_I64_PASS0_I32;
        if (p0) acc_dtype = FHT_I64;
        *plan = create_plan(width, height, strategy, in_dtype, acc_dtype, out_dtype, quadrant_mask, batch, layout,
                            device, p0);
    });
}

int fht_plan_destroy(fht_plan_t plan) {
    return guarded([&] { delete plan; });
}

size_t fht_workspace_bytes(fht_plan_t plan) { return plan ? plan->ws_bytes : 0; }

uint64_t fht_additions(fht_plan_t plan) { return plan ? plan->additions : 0; }

int fht_launches_per_execute(fht_plan_t plan) { return plan ? plan->launches : 0; }

int fht_plan_describe(fht_plan_t plan, char* buf, size_t len) {
    return guarded([&] {
        if (!plan || !buf || !len) throw std::invalid_argument("fht_plan_describe: null argument");
        std::ostringstream o;
        o << "{\"width\":" << plan->w << ",\"height\":" << plan->h << ",\"batch\":" << plan->batch
          << ",\"chunk\":" << plan->chunk << ",\"workspace_bytes\":" << plan->ws_bytes
          << ",\"launches\":" << plan->launches << ",\"additions\":" << plan->additions << ",\"groups\":[";
        for (size_t i = 0; i < plan->groups.size(); ++i) {
            const Group& g = *plan->groups[i];
            o << (i ? "," : "") << "{\"quadrants\":[";
            for (int k = 0; k < g.qs.n; ++k) o << (k ? "," : "") << g.qs.code[k];
            o << "],\"ld\":" << g.ld << ",\"S\":" << g.S << ",\"sr\":" << g.sr << ",\"nbuf\":" << g.nbuf
              << ",\"level_pairs\":" << (g.pairs ? "true" : "false") << ",\"stage_pitch\":" << g.stage_pitch
              << ",\"stage_bytes\":" << g.stage_img << ",\"u16_pair_D\":" << g.pm_D
              << ",\"k2_tma_windows\":"
              << (std::any_of(g.dt.passes.begin(), g.dt.passes.end(), [&](const fhtb::PassDev& d) {
                     return d.tma || (d.ktma && !g.pm_D);
                 }) ? "true" : "false")
              << ",\"pass_rows\":[";
            for (size_t k = 0; k < g.dt.passes.size(); ++k)
                o << (k ? "," : "") << "[" << g.dt.passes[k].S << "," << g.dt.passes[k].L << "]";
            o << "],\"plan\":" << g.sp.describe() << "}";
        }
        o << "]}";
        const std::string s = o.str();
        if (s.size() + 1 > len) throw std::invalid_argument("fht_plan_describe: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

int fht_execute(fht_plan_t plan, const void* d_in, int64_t in_image_stride, void* const d_out[4],
                int64_t out_image_stride, void* d_workspace, void* stream) {
    return guarded([&] {
        if (!plan || !d_out) throw std::invalid_argument("fht_execute: null argument");
        execute(plan, d_in, in_image_stride, d_out, out_image_stride, d_workspace, static_cast<cudaStream_t>(stream));
    });
}

int fht_execute_profiled(fht_plan_t plan, const void* d_in, int64_t in_image_stride, void* const d_out[4],
                         int64_t out_image_stride, void* d_workspace, void* stream, float* launch_ms, int* launch_kind,
                         double* launch_bytes, int max_launches, int* n_launches) {
    struct Ctx {
        cudaStream_t st;
        std::vector<cudaEvent_t> ev;
        std::vector<int> kind;
    };
    Ctx c;
    c.st = static_cast<cudaStream_t>(stream);
    auto hook = [](void* vp, int kind) {
        Ctx* cx = static_cast<Ctx*>(vp);
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, cx->st);
        cx->ev.push_back(e);
        cx->kind.push_back(kind);
    };
    const int rc = guarded([&] {
        if (!plan || !d_out) throw std::invalid_argument("fht_execute_profiled: null argument");
        DeviceGuard dg(plan->device);
        cudaEvent_t e0;
        cuda_check(cudaEventCreate(&e0), "cudaEventCreate");
        cuda_check(cudaEventRecord(e0, c.st), "cudaEventRecord");
        c.ev.push_back(e0);
        c.kind.push_back(0);
        execute(plan, d_in, in_image_stride, d_out, out_image_stride, d_workspace, c.st, hook, &c);
        cuda_check(counted_sync(c.st), "cudaStreamSynchronize");
        const int n = static_cast<int>(c.ev.size()) - 1;
        if (n_launches) *n_launches = n;
        // Algorithmic bytes of each launch (every distinct input
        // cell read once, every output cell written once), in launch order.
        std::vector<double> bytes;
        const double ein = static_cast<double>(esize(plan->in)), ea = static_cast<double>(esize(plan->acc)),
                     eo = static_cast<double>(esize(plan->out));
        for (int img0 = 0; img0 < plan->batch; img0 += plan->chunk) {
            const double nimg = std::min(plan->chunk, plan->batch - img0);
            for (auto& gp : plan->groups) {
                const Group& g = *gp;
                const double slots = nimg * g.qs.n, H = g.sp.H;
                double by_cols = 0, gen_cols = 0;
                for (const auto& b : g.sp.blocks) {
                    const int wdt = g.sp.shapes[static_cast<size_t>(b.shape)].width;
                    (g.use_by32 && !g.sp.root_is_block && wdt == 32 ? by_cols : gen_cols) += wdt;
                }
                // launch order of launch_group: the u8 staging (image read +
                // staged columns written), generic K1, then K1P
                // (u16 pair mode: the pass-0 output cell is 16 bits -- the
                // minimum; the pair layout stores every row twice, which the
                // ncu DRAM traffic shows as overhead)
                const double e0 = g.pm_D ? 2.0 : ea;
                if ((g.nby > 0 || g.pm_D) && g.stage_img > 0)
                    bytes.push_back(nimg * (static_cast<double>(plan->w) * plan->h + static_cast<double>(g.stage_img)));
                if (g.nblocks > 0) bytes.push_back(slots * gen_cols * H * (ein + (g.sp.root_is_block ? eo : e0)));
                if (g.nby > 0) bytes.push_back(slots * by_cols * H * (ein + e0));
                for (size_t k = 0; k < g.sp.passes.size(); ++k)
                    bytes.push_back(slots * g.sp.W * H * ((k == 0 ? e0 : ea) + (k + 1 == g.sp.passes.size() ? eo : ea)));
            }
        }
        for (int i = 0; i < n && i < max_launches && launch_bytes; ++i)
            launch_bytes[i] = i < static_cast<int>(bytes.size()) ? bytes[static_cast<size_t>(i)] : 0.0;
        for (int i = 0; i < n && i < max_launches; ++i) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, c.ev[static_cast<size_t>(i)], c.ev[static_cast<size_t>(i) + 1]),
                       "cudaEventElapsedTime");
            if (launch_ms) launch_ms[i] = ms;
            if (launch_kind) launch_kind[i] = c.kind[static_cast<size_t>(i) + 1];
        }
    });
    for (cudaEvent_t e : c.ev) cudaEventDestroy(e);
    return rc;
}

int fht_execute_pitched(fht_plan_t plan, const void* d_in, int64_t in_row_pitch, int64_t in_image_stride,
                        void* const d_out[4], int64_t out_image_stride, void* d_workspace, void* stream) {
    return guarded([&] {
        if (!plan || !d_out) throw std::invalid_argument("fht_execute_pitched: null argument");
        execute(plan, d_in, in_image_stride, d_out, out_image_stride, d_workspace, static_cast<cudaStream_t>(stream),
                nullptr, nullptr, in_row_pitch);
    });
}

int fht_execute_pitched_peer(fht_plan_t plan, const void* d_in, int64_t in_row_pitch, void* const d_out[4],
                             void* d_workspace, void* d_peer, int peer_first, int peer_end, void* stream) {
    return guarded([&] {
        if (!plan || !d_out) throw std::invalid_argument("fht_execute_pitched_peer: null argument");
        if (plan->layout != FHT_LAYOUT_NATIVE || plan->batch != 1 || plan->groups.size() != 1 ||
            plan->groups[0]->qs.n != 1)
            throw std::invalid_argument("fht_execute_pitched_peer: needs a one-image, one-quadrant, native-layout plan");
        const int W = plan->groups[0]->sp.W;
        if (d_peer && (peer_first < 0 || peer_end > W || peer_first > peer_end))
            throw std::invalid_argument("fht_execute_pitched_peer: bad slope range");
        PeerOut peer;
        peer.ptr = d_peer;
        peer.c0 = peer_first;
        peer.c1 = peer_end;
        execute(plan, d_in, 0, d_out, 0, d_workspace, static_cast<cudaStream_t>(stream), nullptr, nullptr, in_row_pitch,
                0, -1, peer);
    });
}

int fht_device_alloc(size_t bytes, int device, void** d_ptr) {
    return guarded([&] {
        if (!d_ptr) throw std::invalid_argument("fht_device_alloc: null pointer");
        DeviceGuard dg(device);
        cuda_check(counted_malloc(d_ptr, std::max<size_t>(bytes, 1)), "cudaMalloc");
    });
}

int fht_device_free(void* d_ptr) {
    return guarded([&] { cuda_check(cudaFree(d_ptr), "cudaFree"); });
}

int fht_ipc_get_handle(const void* d_ptr, void* handle, size_t handle_len) {
    return guarded([&] {
        if (!d_ptr || !handle || handle_len < sizeof(cudaIpcMemHandle_t))
            throw std::invalid_argument("fht_ipc_get_handle: null pointer or short buffer");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof(h));
    });
}

int fht_ipc_open_handle(const void* handle, size_t handle_len, int device, void** d_ptr) {
    return guarded([&] {
        if (!handle || !d_ptr || handle_len < sizeof(cudaIpcMemHandle_t))
            throw std::invalid_argument("fht_ipc_open_handle: null pointer or short buffer");
        DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        cuda_check(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int fht_ipc_close(void* d_ptr) {
    return guarded([&] { cuda_check(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle"); });
}

int fht_merge_root(int width, int height, int strategy, int acc_dtype, int out_dtype, int layout, const void* d_left,
                   int left_first, const void* d_right, int right_first, int t_begin, int t_end, void* d_out,
                   void* stream) {
    return guarded([&] {
        if (width < 2 || height < 1) throw std::invalid_argument("merge_root: the root must have width >= 2");
        if (!d_left || !d_right || !d_out) throw std::invalid_argument("merge_root: null pointer");
        if (t_begin < 0 || t_end > width || t_begin > t_end) throw std::invalid_argument("merge_root: bad slope range");
        if (layout != FHT_LAYOUT_REFERENCE && layout != FHT_LAYOUT_NATIVE) throw std::invalid_argument("unknown layout");
        if (strategy != FHT_SPLIT_SIMPLE && strategy != FHT_SPLIT_TWEAKED)
            throw std::invalid_argument("unknown strategy (expected simple|tweaked)");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int4* d_ops = merge_root_table(width, height, strategy);
        const int rc = fhtb::launch_merge_root(d_ops, d_left, left_first, d_right, right_first, width, height, t_begin,
                                               t_end, d_out, acc_dtype, out_dtype, layout, st);
        if (rc < 0) throw std::invalid_argument("merge_root: unsupported (accumulator, output) dtype pair");
        cuda_check(cudaGetLastError(), "merge_root launch");
    });
}

int fht_execute_host(fht_plan_t plan, const void* h_in, void* const h_out[4], void* stream) {
    return guarded([&] {
        if (!plan || !h_out) throw std::invalid_argument("fht_execute_host: null argument");
        execute_host(plan, h_in, h_out, static_cast<cudaStream_t>(stream));
    });
}

int fht_check_budget(const void* d_in, int dtype, int64_t count, int width, int* ok_for_i32, void* stream) {
    return guarded([&] { check_budget(d_in, dtype, count, width, ok_for_i32, static_cast<cudaStream_t>(stream)); });
}

int fht_fht2d_counted_i64(const int64_t* img, int width, int height, int strategy, int64_t* hough,
                          uint64_t* additions) {
    return guarded([&] {
        int64_t* outs[4] = {hough, nullptr, nullptr, nullptr};
        run_i64(img, width, height, strategy, FHT_HORIZ_POS, outs, additions);
    });
}

int fht_fht2d_quadrants_i64(const int64_t* img, int width, int height, int strategy, int64_t* horiz_pos,
                            int64_t* horiz_neg, int64_t* vert_pos, int64_t* vert_neg, uint64_t* total_additions) {
    return guarded([&] {
        int64_t* outs[4] = {horiz_pos, horiz_neg, vert_pos, vert_neg};
        run_i64(img, width, height, strategy, FHT_ALL_QUADRANTS, outs, total_additions);
    });
}

int fht_fht2d_pattern(int n, int t, int strategy, int* values) {
    return guarded([&] {
        if (!values) throw std::invalid_argument("fht2d_pattern: null output");
        fhtb::build_pattern(n, t, strategy, values);
    });
}

int fht_slow_hough_device(const void* d_img, int in_dtype, int width, int height, int strategy, int quadrant,
                          int64_t* d_hough, void* stream) {
    return guarded([&] {
        if (!d_img || !d_hough) throw std::invalid_argument("slow_hough: null pointer");
        if (width < 1 || height < 1) throw std::invalid_argument("slow_hough: image is empty");
        if (in_dtype != FHT_U8 && in_dtype != FHT_I32 && in_dtype != FHT_I64)
            throw std::invalid_argument("slow_hough: integer images only");
        if (quadrant < 0 || quadrant > 3) throw std::invalid_argument("slow_hough: quadrant must be 0..3");
        const int W = quadrant < 2 ? width : height, H = quadrant < 2 ? height : width;
        std::vector<int> pat(static_cast<size_t>(W) * W);
        for (int t = 0; t < W; ++t) fhtb::build_pattern(W, t, strategy, pat.data() + static_cast<size_t>(t) * W);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        int* d_pat = nullptr;
        long long* d_cols = nullptr;
        cuda_check(counted_malloc_async(reinterpret_cast<void**>(&d_pat), pat.size() * sizeof(int), st), "cudaMallocAsync");
        cuda_check(counted_malloc_async(reinterpret_cast<void**>(&d_cols), static_cast<size_t>(W) * H * 8, st), "cudaMallocAsync");
        cuda_check(cudaMemcpyAsync(d_pat, pat.data(), pat.size() * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
        fhtb::launch_slow_hough(d_img, in_dtype, width, height, quadrant, d_pat, W, H, d_cols,
                                reinterpret_cast<long long*>(d_hough), st);
        cuda_check(cudaGetLastError(), "slow_hough launch");
        cuda_check(cudaFreeAsync(d_pat, st), "cudaFreeAsync");
        cuda_check(cudaFreeAsync(d_cols, st), "cudaFreeAsync");
        cuda_check(counted_sync(st), "cudaStreamSynchronize");  // the host pattern table goes out of scope
    });
}

int fht_slow_hough_i64(const int64_t* img, int width, int height, int strategy, int64_t* hough) {
    return guarded([&] {
        if (!img || width < 1 || height < 1) throw std::invalid_argument("slow_hough: image is empty");
        cudaStream_t st = cudaStreamPerThread;
        const size_t cells = static_cast<size_t>(width) * height;
        void* d_in = nullptr;
        void* d_out = nullptr;
        cuda_check(counted_malloc_async(&d_in, cells * 8, st), "cudaMallocAsync");
        cuda_check(counted_malloc_async(&d_out, cells * 8, st), "cudaMallocAsync");
        try {
            cuda_check(cudaMemcpyAsync(d_in, img, cells * 8, cudaMemcpyHostToDevice, st), "H2D");
            check_budget(d_in, FHT_I64, static_cast<int64_t>(cells), width, nullptr, st);  // oracle.cpp:11
            const int rc = fht_slow_hough_device(d_in, FHT_I64, width, height, strategy, 0,
                                                 static_cast<int64_t*>(d_out), st);
            if (rc != FHT_OK) throw FhtError(rc, g_last_error);
            cuda_check(cudaMemcpyAsync(hough, d_out, cells * 8, cudaMemcpyDeviceToHost, st), "D2H");
            cuda_check(counted_sync(st), "cudaStreamSynchronize");
        } catch (...) {
            cudaFreeAsync(d_in, st);
            cudaFreeAsync(d_out, st);
            counted_sync(st);
            throw;
        }
        cudaFreeAsync(d_in, st);
        cudaFreeAsync(d_out, st);
        cuda_check(counted_sync(st), "cudaStreamSynchronize");
    });
}

int fht_max_deviation_numerators(int n_lo, int n_hi, int strategy, int64_t* worst) {
    return guarded([&] {
        if (n_lo < 1 || n_hi < n_lo || n_hi > 46340) throw std::invalid_argument("max_deviation: need 1 <= n_lo <= n_hi <= 46340");
        if (strategy != FHT_SPLIT_SIMPLE && strategy != FHT_SPLIT_TWEAKED) throw std::invalid_argument("unknown strategy");
        if (!worst) throw std::invalid_argument("max_deviation: null output");
        const size_t cnt = static_cast<size_t>(n_hi - n_lo + 1);
        cudaStream_t st = cudaStreamPerThread;
        unsigned long long* d = nullptr;
        cuda_check(counted_malloc_async(reinterpret_cast<void**>(&d), cnt * 8, st), "cudaMallocAsync");
        cuda_check(cudaMemsetAsync(d, 0, cnt * 8, st), "cudaMemsetAsync");
        // slices of widths keep each launch's grid.y and run time bounded
        for (int a = n_lo; a <= n_hi; a += 8192) {
            const int b = std::min(n_hi, a + 8191);
            fhtb::launch_max_deviation(a, b, strategy, d + (a - n_lo), st);
        }
        cuda_check(cudaGetLastError(), "max_deviation launch");
        cuda_check(cudaMemcpyAsync(worst, d, cnt * 8, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaFreeAsync(d, st), "cudaFreeAsync");
        cuda_check(counted_sync(st), "cudaStreamSynchronize");
    });
}

int fht_split_width(int w, int strategy, int* w0, int* w1) {
    return guarded([&] {
        if (strategy != FHT_SPLIT_SIMPLE && strategy != FHT_SPLIT_TWEAKED) throw std::invalid_argument("unknown strategy");
        auto pr = fhtb::split_width(w, strategy);
        if (w0) *w0 = pr.first;
        if (w1) *w1 = pr.second;
    });
}

int fht_round_half_up_ratio(int64_t num, int64_t den, int64_t* result) {
    return guarded([&] {
        const int64_t v = fhtb::round_half_up_ratio(num, den);
        if (result) *result = v;
    });
}

int fht_count_additions_tree(int w, int h, int strategy, uint64_t* result) {
    return guarded([&] {
        const uint64_t v = fhtb::count_additions_tree(w, h, strategy);
        if (result) *result = v;
    });
}

int fht_schedule_json(int W, int H, int strategy, int block_width, int pass_levels, int tile_width, char* buf,
                      size_t len, size_t* needed) {
    return guarded([&] {
        const SubPlan sp = SubPlan::build(W, H, strategy, block_width, pass_levels, tile_width);
        std::ostringstream o;
        o << "{\"W\":" << sp.W << ",\"H\":" << sp.H << ",\"root_is_block\":" << (sp.root_is_block ? 1 : 0)
          << ",\"additions\":" << sp.additions << ",\"blocks\":[";
        for (size_t i = 0; i < sp.blocks.size(); ++i)
            o << (i ? "," : "") << "[" << sp.blocks[i].x0 << "," << sp.blocks[i].shape << "," << sp.blocks[i].depth << "]";
        o << "],\"shapes\":[";
        for (size_t i = 0; i < sp.shapes.size(); ++i) {
            const auto& s = sp.shapes[i];
            o << (i ? "," : "") << "{\"width\":" << s.width << ",\"steps\":" << s.depth << ",\"halo\":" << s.halo
              << ",\"step_offset\":[";
            for (size_t k = 0; k < s.step_offset.size(); ++k) o << (k ? "," : "") << s.step_offset[k];
            o << "],\"ops\":[";
            for (size_t k = 0; k < s.ops.size(); ++k)
                o << (k ? "," : "") << "[" << s.ops[k].dst << "," << s.ops[k].a << "," << s.ops[k].b << "," << s.ops[k].r
                  << "," << s.extra[k] << "]";
            o << "]}";
        }
        o << "],\"passes\":[";
        for (size_t i = 0; i < sp.passes.size(); ++i) {
            const auto& ps = sp.passes[i];
            o << (i ? "," : "") << "{\"levels\":" << ps.levels << ",\"max_slots\":" << ps.max_slots
              << ",\"max_ext\":" << ps.max_ext << ",\"tiles\":[";
            for (size_t k = 0; k < ps.tiles.size(); ++k) {
                const auto& t = ps.tiles[k];
                o << (k ? "," : "") << "[" << t.load_beg << "," << t.load_cnt << "," << t.step_beg << "," << t.nsteps << ","
                  << t.store_beg << "," << t.store_cnt << "," << t.nslots << "," << t.max_ext << "]";
            }
            o << "],\"loads\":[";
            for (size_t k = 0; k < ps.loads.size(); ++k)
                o << (k ? "," : "") << "[" << ps.loads[k].gcol << "," << ps.loads[k].slot << "," << ps.loads[k].off << ","
                  << ps.loads[k].ext << "]";
            o << "],\"step_offs\":[";
            for (size_t k = 0; k < ps.step_offs.size(); ++k) o << (k ? "," : "") << ps.step_offs[k];
            o << "],\"ops\":[";
            for (size_t k = 0; k < ps.ops.size(); ++k) {
                const auto& op = ps.ops[k];
                o << (k ? "," : "") << "[" << op.dst << "," << op.a << "," << op.b << "," << op.ad << "," << op.bd << ","
                  << op.ext << "]";
            }
            o << "],\"stores\":[";
            for (size_t k = 0; k < ps.stores.size(); ++k)
                o << (k ? "," : "") << "[" << ps.stores[k].slot << "," << ps.stores[k].gcol << "]";
            // the level-pair program (ops: [dst, ext, [[slot, off], ...]])
            o << "],\"pairs\":{\"max_slots\":" << ps.pmax_slots << ",\"tiles\":[";
            for (size_t k = 0; k < ps.ptiles.size(); ++k) {
                const auto& t = ps.ptiles[k];
                o << (k ? "," : "") << "[" << t.load_beg << "," << t.load_cnt << "," << t.step_beg << "," << t.nsteps << ","
                  << t.store_beg << "," << t.store_cnt << "," << t.nslots << "," << t.max_ext << "]";
            }
            o << "],\"step_offs\":[";
            for (size_t k = 0; k < ps.pstep_offs.size(); ++k) o << (k ? "," : "") << ps.pstep_offs[k];
            o << "],\"ops\":[";
            for (size_t k = 0; k < ps.pops.size(); ++k) {
                const auto& op = ps.pops[k];
                o << (k ? "," : "") << "[" << op.dst << "," << op.ext << ",[";
                for (int j = 0; j < op.nterms; ++j)
                    o << (j ? "," : "") << "[" << op.term[j].slot << "," << op.term[j].off << "]";
                o << "]," << op.split << "]";
            }
            o << "],\"stores\":[";
            for (size_t k = 0; k < ps.pstores.size(); ++k)
                o << (k ? "," : "") << "[" << ps.pstores[k].slot << "," << ps.pstores[k].gcol << "]";
            o << "]}}";
        }
        o << "]}";
        const std::string s = o.str();
        if (needed) *needed = s.size() + 1;
        if (!buf || s.size() + 1 > len) throw std::invalid_argument("fht_schedule_json: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

const char* fht_last_error(void) { return g_last_error.c_str(); }

int fht_plan_cache_clear(size_t* released) {
    return guarded([&] {
        const size_t n = plan_cache_clear();
        if (released) *released = n;
    });
}

size_t fht_plan_cache_size(void) { return plan_cache_size(); }

int fht_debug_counters(uint64_t* host_syncs, uint64_t* device_allocs) {
    if (host_syncs) *host_syncs = g_host_syncs.load();
    if (device_allocs) *device_allocs = g_device_allocs.load();
    return FHT_OK;
}

const char* fht_version(void) { return "fht_b200 0.1 (sm_100a)"; }

}  // extern "C"
