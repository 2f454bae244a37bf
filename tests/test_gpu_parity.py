"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle.

Bar: bit-exact for integer inputs; for float32, bit-exact against the fp32
restatement of the same add tree AND max |J - J64| <= 1e-5 * L1 (L1 = the
fp64 transform of |I|), the tolerance BASELINE.json states.
"""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht, workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

Q = oracle.QUADRANTS


def run_plan(imgs, in_dtype, acc, strategy=1, quadrants="all", layout="reference", out_dtype=None):
    imgs = np.ascontiguousarray(imgs)
    if imgs.ndim == 2:
        imgs = imgs[None]
    b, h, w = imgs.shape
    plan = fht.Plan(w, h, strategy, in_dtype=in_dtype, acc_dtype=acc, out_dtype=out_dtype, quadrants=quadrants,
                    batch=b, layout=layout)
    x = torch.from_numpy(imgs).cuda()
    out = plan(x)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}, plan


# ------------------------------------------------- reference entry points
def test_golden_vectors_through_c_abi(golden):
    for row in golden["meta"]:
        i, h, w, strat, adds, qadds = (int(v) for v in row)
        img = golden[f"c{i}_img"].astype(np.int64)
        ct = fht.fht2d_counted(img, strat)
        np.testing.assert_array_equal(ct.hough, golden[f"c{i}_s{strat}_fht2d"])
        assert ct.additions == adds
        tot = []
        qs = fht.fht2d_quadrants(img, strat, tot)
        assert tot == [qadds]
        for k in Q:
            np.testing.assert_array_equal(getattr(qs, k), golden[f"c{i}_s{strat}_{k}"])


def test_spec_2x2_and_identity():
    a, b, c, d = 3, 5, 7, 11
    j = fht.fht2d(np.array([[a, b], [c, d]]), "tweaked")
    assert j[0, 0] == a + b and j[1, 0] == c + d and j[0, 1] == a + d and j[1, 1] == c + b
    col = np.arange(9).reshape(9, 1)
    np.testing.assert_array_equal(fht.fht2d(col), col)  # w = 1 -> identity
    assert fht.fht2d_counted(col).additions == 0


def test_int64_values_use_int64_accumulation():
    rng = np.random.default_rng(11)
    img = rng.integers(-(1 << 40), 1 << 40, (37, 53))
    for s in (0, 1):
        np.testing.assert_array_equal(fht.fht2d(img, s), oracle.fht2d_counted_i64(img, s)[0])


@pytest.mark.parametrize("ind", ["i32", "i64"])
def test_int64_plan_with_int32_pass0(ind):
    """acc i64 with pass 0 in int32 (FHT_I64_PASS0_I32): values whose full
    sums need int64 (W * max|v| >= 2^31) but whose width-32 blocks fit int32
    (32 * max|v| < 2^31) -- identical to the all-int64 plan and the oracle."""
    rng = np.random.default_rng(12)
    h, w = 301, 1000
    imgs = rng.integers(-(1 << 25), 1 << 25, (2, h, w)).astype({"i32": np.int32, "i64": np.int64}[ind])
    x = torch.from_numpy(imgs).cuda()
    mixed = fht.Plan(w, h, 1, in_dtype=ind, acc_dtype="i64", batch=2, pass0_i32=True)(x)
    full = fht.Plan(w, h, 1, in_dtype=ind, acc_dtype="i64", batch=2)(x)
    torch.cuda.synchronize()
    for b in range(2):
        ref, _ = oracle.fht2d_quadrants(imgs[b].astype(np.int64), 1, dtype=np.int64)
        for k in Q:
            np.testing.assert_array_equal(mixed[k][b].cpu().numpy(), ref[k])
            np.testing.assert_array_equal(full[k][b].cpu().numpy(), ref[k])


def test_int64_entry_points_choose_int32_pass0():
    """fht2d_counted / fht2d_quadrants on values in [2^31 / W, 2^26): the
    entry point picks the int64 plan with pass 0 in int32; bit-exact."""
    rng = np.random.default_rng(13)
    img = rng.integers(-(1 << 24), 1 << 24, (257, 700))
    for s in (0, 1):
        r = fht.fht2d_counted(img, s)
        ref, adds = oracle.fht2d_counted_i64(img, s)
        np.testing.assert_array_equal(r.hough, ref)
        assert r.additions == adds
    q = fht.fht2d_quadrants(img, 1)
    refq, _ = oracle.fht2d_quadrants(img, 1, dtype=np.int64)
    for k in Q:
        np.testing.assert_array_equal(getattr(q, k), refq[k])


def test_errors_mirror_reference():
    with pytest.raises(fht.OverflowBudget):
        fht.fht2d(np.full((3, 4), 1 << 61, dtype=np.int64))
    with pytest.raises(fht.InvalidArgument):
        fht.fht2d(np.zeros((0, 4), dtype=np.int64))
    with pytest.raises(fht.InvalidArgument):
        fht.fht2d(np.zeros((2, 2), dtype=np.int64), 7)
    with pytest.raises(fht.InvalidArgument):
        fht.Plan(0, 5)
    with pytest.raises(fht.OverflowBudget):
        fht.Plan(9_000_000, 1, in_dtype="u8", acc_dtype="i32", quadrants="horiz_pos")


# ---------------------------------------------------------- plan API
@pytest.mark.parametrize("strategy", [0, 1])
def test_small_sizes_all_quadrants_batched(strategy):
    rng = np.random.default_rng(100 + strategy)
    for (h, w) in [(1, 1), (1, 9), (9, 1), (2, 2), (3, 5), (17, 17), (31, 33), (33, 31), (40, 64), (64, 40),
                   (65, 65), (100, 7), (7, 100), (129, 130)]:
        imgs = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
        out, plan = run_plan(imgs, "u8", "i32", strategy)
        for bi in range(3):
            ref, adds = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
            for k in Q:
                np.testing.assert_array_equal(out[k][bi], ref[k], err_msg=f"{h}x{w} {k} img{bi}")
        assert plan.additions == 3 * adds


def test_native_layout_and_widening():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (45, 77), dtype=np.uint8)
    ref, _ = oracle.fht2d_quadrants(img, 1)
    out, _ = run_plan(img, "u8", "i32", layout="native")
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k].T)
    out, _ = run_plan(img, "u8", "i32", out_dtype="i64")
    for k in Q:
        assert out[k].dtype == np.int64
        np.testing.assert_array_equal(out[k][0], ref[k])
    out, _ = run_plan(img, "u8", "i64")
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k])


def test_int32_inputs_with_negative_values():
    rng = np.random.default_rng(6)
    img = rng.integers(-(1 << 20), 1 << 20, (70, 90)).astype(np.int32)
    out, _ = run_plan(img, "i32", "i32", strategy=0)
    ref, _ = oracle.fht2d_quadrants(img, 0, dtype=np.int32)
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k])


def test_float32_small_bit_exact_vs_fp32_tree():
    rng = np.random.default_rng(8)
    for (h, w) in [(37, 53), (64, 64), (200, 131)]:
        img = rng.standard_normal((h, w)).astype(np.float32)
        out, _ = run_plan(img, "f32", "f32")
        ref, _ = oracle.fht2d_quadrants(img, 1, dtype=np.float32)
        for k in Q:
            np.testing.assert_array_equal(out[k][0], ref[k])


@pytest.mark.parametrize("k1p,k2,pairs,bulk,stage", [(0, 0, 0, 0, 0), (2, 0, 0, 0, 1), (2, 1, 0, 0, 0), (3, 0, 0, 1, 1), (4, 1, 1, 0, 1), (4, 0, 0, 0, 0),
                                                    (3, 1, 0, 0, 0), (3, 1, 1, 0, 1), (3, 1, 1, 1, 0), (0, 1, 1, 0, 1), (5, 1, 1, 0, 1), (5, 1, 1, 0, 0)])
def test_kernel_variants_bit_exact(monkeypatch, k1p, k2, pairs, bulk, stage):
    """Every K1P level variant (0: all levels in shared memory, 2: levels 1-2
    in registers, 3: + interleaved levels 3-5), both one-level K2 merge
    layouts (0: 4 rows per lane, 1: rows interleaved over lanes), the
    level-pair K2 programs and the TMA bulk window loads, against the oracle
    (the f32 case bit-exact: pairs keep the tree's add order)."""
    monkeypatch.setenv("FHT_K1P_VARIANT", str(k1p))
    monkeypatch.setenv("FHT_K2_SCALAR", str(k2))
    monkeypatch.setenv("FHT_K2_PAIRS", str(pairs))
    monkeypatch.setenv("FHT_K2_BULK", str(bulk))
    monkeypatch.setenv("FHT_K1_STAGE", str(stage))  # u8 images staged as aligned columns for K1P
    rng = np.random.default_rng(40 + 10 * k1p + k2)
    for strategy, (h, w) in [(1, (509, 509)), (0, (300, 257)), (1, (1000, 70))]:
        imgs = rng.integers(0, 256, (2, h, w), dtype=np.uint8)
        out, _ = run_plan(imgs, "u8", "i32", strategy)
        for bi in range(2):
            ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
            for k in Q:
                np.testing.assert_array_equal(out[k][bi], ref[k], err_msg=f"{h}x{w} s{strategy} {k}")
    img = rng.standard_normal((333, 271)).astype(np.float32)
    out, _ = run_plan(img, "f32", "f32")
    ref, _ = oracle.fht2d_quadrants(img, 1, dtype=np.float32)
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k])


@pytest.mark.parametrize("k576", [0, 1])
@pytest.mark.parametrize("ind,acc", [("u8", "i32"), ("i32", "i32"), ("f32", "f32")])
def test_k1p_thread_counts(monkeypatch, k576, ind, acc):
    """K1P variant 5 on 576 threads (one round of level-1/2 items; warps 16-17
    only in those levels) and on 512, unstaged, with full and partial row tiles."""
    monkeypatch.setenv("FHT_K1P_576", str(k576))
    monkeypatch.setenv("FHT_K1_STAGE", "0")
    rng = np.random.default_rng(7 + k576)
    for strategy, (h, w) in [(1, (600, 333)), (0, (257, 96))]:
        if ind == "f32":
            img = rng.standard_normal((h, w)).astype(np.float32)
        else:
            img = rng.integers(-100 if ind == "i32" else 0, 256, (h, w)).astype(np.uint8 if ind == "u8" else np.int32)
        out, _ = run_plan(img, ind, acc, strategy)
        ref, _ = oracle.fht2d_quadrants(img, strategy, dtype=np.float32 if ind == "f32" else np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][0], ref[k], err_msg=f"{h}x{w} s{strategy} {k}")


# --------------------------------------------------- the five configs
def _cfg_plan(cfg, count=None):
    c = workloads.CONFIGS[cfg]
    imgs = workloads.make_images(cfg, count)
    out, plan = run_plan(imgs, c.dtype, c.acc, 1, quadrants=list(c.quadrants))
    return c, imgs, out, plan


def test_config_c1_bit_exact():
    c, imgs, out, plan = _cfg_plan("c1")
    ref, adds = oracle.fht2d(imgs[0].T, 1, dtype=np.int32)  # vert_pos = fht2d(I^T)
    np.testing.assert_array_equal(out["vert_pos"][0], ref)
    assert plan.additions == adds == 9_984_000
    # the reference's own fht2d(I) family (horiz_pos) as a parity extra
    out2, _ = run_plan(imgs, "u8", "i32", 1, quadrants="horiz_pos")
    np.testing.assert_array_equal(out2["horiz_pos"][0], oracle.fht2d(imgs[0], 1, dtype=np.int32)[0])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref (the compiled reference) not built")
def test_configs_c1_c2_against_compiled_reference():
    """Full-size parity against the reference library itself (not the port):
    c1 = vert_pos = fht::fht2d(transpose(I)) (transform.cpp:62-89), c2 = the
    four quadrants of fht::fht2d_quadrants (quadrants.cpp:23-41), int64."""
    c, imgs, out, _ = _cfg_plan("c1")
    ref, adds = oracle.ref_fht2d_counted(np.ascontiguousarray(imgs[0].T))
    np.testing.assert_array_equal(out["vert_pos"][0], ref)
    assert adds == 9_984_000
    c, imgs, out, _ = _cfg_plan("c2")
    ref, adds = oracle.ref_fht2d_quadrants(imgs[0])
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k])
    assert adds == 4 * 10_485_760
    # and the int64 drop-in entry point on the same image
    tot = []
    qs = fht.fht2d_quadrants(imgs[0].astype(np.int64), "tweaked", tot)
    for k in Q:
        np.testing.assert_array_equal(getattr(qs, k), ref[k])
    assert tot == [adds]


def test_config_c2_bit_exact_and_strategies_coincide():
    c, imgs, out, plan = _cfg_plan("c2")
    ref, adds = oracle.fht2d_quadrants(imgs[0], 1, dtype=np.int32)
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k])
    assert plan.additions == adds == 4 * 10_485_760
    out_s, _ = run_plan(imgs, "u8", "i32", 0)
    for k in Q:
        np.testing.assert_array_equal(out_s[k], out[k])  # Simple == Tweaked at n = 2^q


def _float_check(img, out, quadrant):
    """bit-exact vs the fp32 tree and within 1e-5 * L1 of the fp64 tree."""
    src = {"horiz_pos": img, "horiz_neg": img[:, ::-1], "vert_pos": img.T, "vert_neg": img.T[:, ::-1]}[quadrant]
    src = np.ascontiguousarray(src)
    j32, _ = oracle.fht2d(src, 1, dtype=np.float32)
    np.testing.assert_array_equal(out, j32)
    j64, _ = oracle.fht2d(src.astype(np.float64), 1, dtype=np.float64)
    l1, _ = oracle.fht2d(np.abs(src).astype(np.float64), 1, dtype=np.float64)
    err = np.abs(out.astype(np.float64) - j64) / l1
    assert err.max() <= 1e-5, err.max()


def test_config_c3_float32():
    c, imgs, out, plan = _cfg_plan("c3")
    for k in Q:
        _float_check(imgs[0], out[k][0], k)


def test_config_c4_batch():
    c, imgs, out, plan = _cfg_plan("c4")
    assert out["horiz_pos"].shape == (256, 509, 509)
    rng = np.random.default_rng(0)
    for bi in sorted(rng.choice(256, 24, replace=False)):  # full oracle compare on a seeded sample
        ref, _ = oracle.fht2d_quadrants(imgs[bi], 1, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][bi], ref[k])
    if oracle.ref_available():
        # all 256 images x 4 quadrants against the compiled reference itself
        # (fht::fht2d_quadrants, quadrants.cpp:23-41, on the host threads)
        for b0 in range(0, 256, 32):
            ref = oracle.ref_batch_quadrants_u8(imgs[b0:b0 + 32], 1, threads=oracle.host_threads(),
                                                want_output=True)
            for qi, k in enumerate(Q):
                got = out[k][b0:b0 + 32].reshape(32, -1)
                assert np.array_equal(got, ref[:, qi]), (b0, k)
    # every image: mass conservation per slope, a size-independent property
    mass = imgs.reshape(256, -1).sum(axis=1).astype(np.int64)
    for k in Q:
        col = out[k].astype(np.int64).sum(axis=1)  # sum over s -> (256, W)
        assert (col == mass[:, None]).all()


def test_config_c5_float32():
    c, imgs, out, plan = _cfg_plan("c5")
    img = imgs[0]
    for k in Q:  # all four quadrants against the full fp32 and fp64 trees (~10 s each)
        _float_check(img, out[k][0], k)
    tot = float(img.astype(np.float64).sum())
    for k in Q:  # all four: mass conservation within fp32 rounding
        col = out[k][0].astype(np.float64).sum(axis=0)
        assert np.allclose(col, tot, rtol=1e-4)


def test_shift_equivariance_and_linearity_large():
    rng = np.random.default_rng(9)
    n = 1000
    a = rng.integers(0, 100, (n, n), dtype=np.int32)
    b = rng.integers(0, 100, (n, n), dtype=np.int32)
    ja, _ = run_plan(a, "i32", "i32")
    jb, _ = run_plan(b, "i32", "i32")
    jab, _ = run_plan(3 * a + 2 * b, "i32", "i32")
    for k in Q:
        np.testing.assert_array_equal(jab[k], 3 * ja[k] + 2 * jb[k])
    r = 37
    jr, _ = run_plan(np.roll(a, -r, axis=0), "i32", "i32", quadrants="horiz_pos")
    np.testing.assert_array_equal(jr["horiz_pos"][0], np.roll(ja["horiz_pos"][0], -r, axis=0))


def test_execute_host_roundtrip():
    rng = np.random.default_rng(12)
    imgs = rng.integers(0, 256, (4, 61, 67), dtype=np.uint8)
    plan = fht.Plan(67, 61, 1, in_dtype="u8", acc_dtype="i32", batch=4)
    out = plan.execute_host(imgs)
    for bi in range(4):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], 1, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][bi], ref[k])


@pytest.mark.parametrize("stage,parts,chunk", [(1, 3, None), (1, 1, 5), (0, 4, 3)])
def test_execute_host_parts_and_chunks(monkeypatch, stage, parts, chunk):
    """The host-buffer path cuts a batch into parts on three streams, each with
    its own workspace slice; with u8 staging the staged columns live after a
    chunk's slot buffers.  Every image must match the oracle (and the device
    path) whatever the part/chunk split."""
    monkeypatch.setenv("FHT_K1_STAGE", str(stage))
    monkeypatch.setenv("FHT_HOST_PARTS", str(parts))
    if chunk:
        monkeypatch.setenv("FHT_CHUNK_IMAGES", str(chunk))
    rng = np.random.default_rng(13)
    n, b = 509, 11
    imgs = rng.integers(0, 256, (b, n, n), dtype=np.uint8)
    plan = fht.Plan(n, n, 1, in_dtype="u8", acc_dtype="i32", batch=b)
    assert (plan.describe()["groups"][0]["stage_bytes"] > 0) == bool(stage)
    host = plan.execute_host(imgs)
    dev, _ = run_plan(imgs, "u8", "i32", 1)
    for bi in (0, 4, b - 1):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], 1, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(host[k][bi], ref[k], err_msg=f"host img{bi} {k}")
    for k in Q:
        np.testing.assert_array_equal(host[k], dev[k])


def test_profiled_launch_accounting(monkeypatch):
    """fht_execute_profiled: one record per launch, kinds in launch order and
    algorithmic bytes that add up to the plan's passes (bench roofline input)."""
    import ctypes

    from paper_2411_07351_b200._lib import check, lib

    n = 509
    monkeypatch.setenv("FHT_K1_STAGE", "1")  # staged even for this small batch
    plan = fht.Plan(n, n, "tweaked", in_dtype="u8", acc_dtype="i32", batch=3)
    x = torch.zeros((3, n, n), dtype=torch.uint8, device="cuda")
    out = plan.alloc_outputs()
    ptrs = (ctypes.c_void_p * 4)(*[out[q].data_ptr() for q in fht.QUADRANTS])
    ws = plan.workspace()
    nl = plan.launches
    ms, kind, by, got = (ctypes.c_float * nl)(), (ctypes.c_int * nl)(), (ctypes.c_double * nl)(), ctypes.c_int()
    check(lib().fht_execute_profiled(plan._h, ctypes.c_void_p(x.data_ptr()), n * n, ptrs, n * n,
                                     ctypes.c_void_p(ws.data_ptr()), None, ms, kind, by, nl, ctypes.byref(got)))
    assert got.value == nl == 4
    kinds, b = list(kind), list(by)
    # u8 staging of the horizontal (T) and vertical (P) working columns,
    # generic K1 (remainder block), K1P, root band
    assert kinds == [5, 1, 4, 3]
    slots, cells = 3 * 4, n * n
    # the u16 pair mode is on for 509^2 u8: pass-0 cells are 16 bits
    assert plan.describe()["groups"][0]["u16_pair_D"] == 256
    assert b[1] + b[2] == slots * cells * (1 + 2)  # pass 0 covers every column once: e_in + e_pass0
    assert b[2] == slots * (n // 32) * 32 * n * 3  # the 15 width-32 blocks
    assert b[3] == slots * cells * (2 + 4)  # u16 cells in, int32 out
    pitch = plan.describe()["groups"][0]["stage_pitch"]
    assert pitch % 16 == 0 and pitch >= n + 31
    assert b[0] == 3 * (cells + 2 * n * pitch)  # image read + both staged column sets written


@pytest.mark.parametrize("h,w,dt", [(300, 777, "f32"), (1000, 1000, "u8"), (96, 3001, "f32"), (513, 130, "i32")])
def test_tma_band_windows_option(monkeypatch, h, w, dt):
    """FHT_K2_TMA_BANDS=1: the level-pair bands' windows by the TMA engine,
    alignment residues applied per row tile at run time -- bit-exact."""
    rng = np.random.default_rng(h + w)
    img = (rng.standard_normal((h, w)).astype(np.float32) if dt == "f32"
           else rng.integers(0, 200, (h, w)).astype(np.uint8 if dt == "u8" else np.int32))
    acc = "f32" if dt == "f32" else "i32"
    monkeypatch.setenv("FHT_K2_TMA_BANDS", "1")
    out, plan = run_plan(img, dt, acc)
    assert any(g["k2_tma_windows"] for g in plan.describe()["groups"])
    ref, _ = oracle.fht2d_quadrants(img, 1, dtype=np.float32 if dt == "f32" else np.int32)
    for k in Q:
        np.testing.assert_array_equal(out[k][0], ref[k])
