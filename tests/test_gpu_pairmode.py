"""GPU parity of the u16 pair mode: u8 images whose root
children are at most 257 wide run with 32-bit words holding rows j and
j + D, the root step widening to int32.  Bit-exact against the oracle at the
shape limits, for worst-case (all-255) images, odd and even heights, both
strategies, int64 output, the native layout and single quadrants; and
against the mode switched off (FHT_U16_PAIRS=0)."""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

Q = oracle.QUADRANTS


def _run(imgs, strategy=1, quadrants="all", layout="reference", out_dtype=None):
    b, h, w = imgs.shape
    plan = fht.Plan(w, h, strategy, in_dtype="u8", acc_dtype="i32", out_dtype=out_dtype, quadrants=quadrants,
                    batch=b, layout=layout)
    out = plan(torch.from_numpy(np.ascontiguousarray(imgs)).cuda())
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}, plan.describe()


def _pair_d(desc):
    return [g["u16_pair_D"] for g in desc["groups"]]


@pytest.mark.parametrize("h,w,strategy", [(509, 509, 1), (512, 512, 1), (64, 65, 1), (65, 300, 0), (511, 96, 1),
                                          (120, 258, 0), (130, 257, 1), (333, 77, 0)])
def test_pair_mode_bit_exact(h, w, strategy):
    rng = np.random.default_rng(h * 1000 + w)
    imgs = rng.integers(0, 256, (2, h, w), dtype=np.uint8)
    imgs[1] = 255  # the overflow worst case: every node sum at its bound
    out, desc = _run(imgs, strategy)
    assert any(d > 0 for d in _pair_d(desc)), desc
    for bi in range(2):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][bi], ref[k], err_msg=f"{h}x{w} s{strategy} {k} img{bi}")


def test_pair_mode_off_beyond_limits():
    # root children of 514 (Tweaked: 256 + 258) exceed 257: the mode stays off
    _, desc = _run(np.zeros((1, 100, 514), np.uint8), 1, quadrants="horiz_pos")
    assert _pair_d(desc) == [0]
    # H > 512: D would exceed one 256-word tile
    _, desc = _run(np.zeros((1, 513, 300), np.uint8), 1, quadrants="horiz_pos")
    assert _pair_d(desc) == [0]


def test_pair_mode_layouts_widening_quadrants(monkeypatch):
    rng = np.random.default_rng(7)
    imgs = rng.integers(0, 256, (3, 300, 420), dtype=np.uint8)
    ref = [oracle.fht2d_quadrants(imgs[i], 1, dtype=np.int64)[0] for i in range(3)]
    out, desc = _run(imgs, 1, out_dtype="i64")
    assert all(d > 0 for d in _pair_d(desc))
    for i in range(3):
        for k in Q:
            assert out[k].dtype == np.int64
            np.testing.assert_array_equal(out[k][i], ref[i][k])
    out, _ = _run(imgs, 1, layout="native")
    for i in range(3):
        for k in Q:
            np.testing.assert_array_equal(out[k][i], ref[i][k].T)
    for q in ("vert_neg", "horiz_pos"):
        out, _ = _run(imgs, 1, quadrants=q)
        for i in range(3):
            np.testing.assert_array_equal(out[q][i], ref[i][q])
    # the same bytes with the mode switched off
    monkeypatch.setenv("FHT_U16_PAIRS", "0")
    out0, desc0 = _run(imgs, 1)
    assert _pair_d(desc0) == [0, 0]
    for i in range(3):
        for k in Q:
            np.testing.assert_array_equal(out0[k][i], ref[i][k])


def test_pair_mode_host_buffers():
    rng = np.random.default_rng(3)
    imgs = rng.integers(0, 256, (5, 509, 509), dtype=np.uint8)
    plan = fht.Plan(509, 509, 1, in_dtype="u8", acc_dtype="i32", quadrants="all", batch=5)
    out = plan.execute_host(imgs)
    for i in (0, 4):
        ref, _ = oracle.fht2d_quadrants(imgs[i], 1, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][i], ref[k])



@pytest.mark.parametrize("bulk", [0, 1])
def test_pair_mode_bulk_windows(monkeypatch, bulk):
    """The pair-mode root band with its windows by cp.async or by TMA bulk copies."""
    monkeypatch.setenv("FHT_K2_BULK", str(bulk))
    rng = np.random.default_rng(10 + bulk)
    imgs = rng.integers(0, 256, (5, 250, 333), dtype=np.uint8)
    out, desc = _run(imgs, 1)
    assert all(d > 0 for d in _pair_d(desc))
    for i in (0, 2, 4):
        ref, _ = oracle.fht2d_quadrants(imgs[i], 1, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][i], ref[k], err_msg=f"img{i} {k}")


@pytest.mark.parametrize("pipe,spc", [(1, 1), (1, 3), (1, 64), (0, 4)])
def test_pair_mode_double_buffered_root_band(monkeypatch, pipe, spc):
    """k2_pair_pipe: each CTA walks `spc` slots with the next slot's windows
    streaming into the second buffer (FHT_K2_PIPE=0: one slot per CTA)."""
    monkeypatch.setenv("FHT_K2_PIPE", str(pipe))
    monkeypatch.setenv("FHT_K2_SLOTS_PER_CTA", str(spc))
    rng = np.random.default_rng(100 + spc)
    imgs = rng.integers(0, 256, (7, 509, 509), dtype=np.uint8)
    imgs[3] = 255
    out, desc = _run(imgs, 1)
    assert _pair_d(desc) == [256]
    for i in (0, 3, 5, 6):
        ref, _ = oracle.fht2d_quadrants(imgs[i], 1, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][i], ref[k], err_msg=f"img{i} {k}")


@pytest.mark.parametrize("k576", [0, 1])
def test_pair_mode_k1p_thread_counts(monkeypatch, k576):
    """The pair mode's K1P on 576 threads (one round of level-1/2 items) and on
    the 512-thread kernel, for odd and even heights."""
    monkeypatch.setenv("FHT_K1P_PAIR576", str(k576))
    rng = np.random.default_rng(5 + k576)
    for h, w in [(509, 509), (400, 256), (129, 300)]:
        imgs = rng.integers(0, 256, (2, h, w), dtype=np.uint8)
        out, desc = _run(imgs, 1)
        assert all(d > 0 for d in _pair_d(desc))
        for i in range(2):
            ref, _ = oracle.fht2d_quadrants(imgs[i], 1, dtype=np.int32)
            for k in Q:
                np.testing.assert_array_equal(out[k][i], ref[k], err_msg=f"{h}x{w} img{i} {k}")


def test_pair_mode_chunks_and_graph_replay(monkeypatch):
    """Pair mode over image chunks (FHT_CHUNK_IMAGES: per-chunk staging and
    slot offsets) and replayed from a captured CUDA graph."""
    monkeypatch.setenv("FHT_CHUNK_IMAGES", "3")
    rng = np.random.default_rng(21)
    imgs = rng.integers(0, 256, (7, 509, 509), dtype=np.uint8)
    plan = fht.Plan(509, 509, 1, in_dtype="u8", acc_dtype="i32", quadrants="all", batch=7)
    assert plan.describe()["chunk"] == 3
    x = torch.from_numpy(imgs).cuda()
    out = plan.alloc_outputs()
    plan(x, out)
    torch.cuda.synchronize()
    refs = {i: oracle.fht2d_quadrants(imgs[i], 1, dtype=np.int32)[0] for i in (0, 3, 6)}
    for i, ref in refs.items():
        for k in Q:
            np.testing.assert_array_equal(out[k][i].cpu().numpy(), ref[k], err_msg=f"chunked img{i} {k}")
    for v in out.values():
        v.zero_()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan(x, out, stream=s)
    g.replay()
    torch.cuda.synchronize()
    for i, ref in refs.items():
        for k in Q:
            np.testing.assert_array_equal(out[k][i].cpu().numpy(), ref[k], err_msg=f"graph img{i} {k}")


@pytest.mark.parametrize("h,w,strategy", [(509, 509, 1), (512, 512, 1), (64, 65, 1), (65, 300, 0), (130, 257, 1),
                                          (333, 77, 0), (257, 511, 1)])
def test_tma_windows_match_cp_async_windows(monkeypatch, h, w, strategy):
    """The pair-mode root band's windows by the TMA engine (bulk copies, the
    window starts aligned down and the residue folded into the ops) against
    the same band with 4/16-byte cp.async windows, and both against the oracle."""
    rng = np.random.default_rng(h + 7 * w)
    imgs = rng.integers(0, 256, (9, h, w), dtype=np.uint8)
    imgs[3] = 255
    out, desc = _run(imgs, strategy)
    assert any(g["k2_tma_windows"] for g in desc["groups"]), desc
    monkeypatch.setenv("FHT_K2_TMA", "0")
    out0, desc0 = _run(imgs, strategy)
    assert not any(g["k2_tma_windows"] for g in desc0["groups"])
    for k in Q:
        np.testing.assert_array_equal(out[k], out0[k])
    for bi in (0, 3, 8):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
        for k in Q:
            np.testing.assert_array_equal(out[k][bi], ref[k], err_msg=f"{h}x{w} {k} img{bi}")


@pytest.mark.parametrize("h,w,strategy", [(509, 509, 1), (65, 300, 0), (257, 511, 1), (100, 300, 1)])
def test_wide_root_band_tiles(monkeypatch, h, w, strategy):
    """32-slope root-band tiles on the 1024-thread pair kernel (an option:
    FHT_TILE_WIDTH=32 with the shared-memory budget raised), TMA windows on
    and off, against the oracle."""
    rng = np.random.default_rng(h * 3 + w)
    imgs = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
    imgs[1] = 255
    monkeypatch.setenv("FHT_TILE_WIDTH", "32")
    monkeypatch.setenv("FHT_K2_SMEM_KB", "125")
    for tma in ("1", "0"):
        monkeypatch.setenv("FHT_K2_TMA", tma)
        out, desc = _run(imgs, strategy)
        for bi in range(3):
            ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
            for k in Q:
                np.testing.assert_array_equal(out[k][bi], ref[k], err_msg=f"{h}x{w} tma{tma} {k} img{bi}")


@pytest.mark.parametrize("seed", range(4))
def test_pair_mode_random_shapes(seed):
    """Seeded random pair-mode shapes (65..512 wide, 64..512 high), both
    strategies, random batches and quadrant masks, some all-255 images (the
    16-bit limit): bit-exact against the oracle (scripts/pair_sweep.py runs
    the same sweep at length)."""
    rng = np.random.default_rng(4000 + seed)
    for _ in range(15):
        w, h = int(rng.integers(65, 513)), int(rng.integers(64, 513))
        strategy, b, mask = int(rng.integers(2)), int(rng.integers(1, 4)), int(rng.integers(1, 16))
        quads = [q for i, q in enumerate(oracle.QUADRANTS) if mask & (1 << i)]
        imgs = rng.integers(0, 256, (b, h, w)).astype(np.uint8)
        if rng.random() < 0.2:
            imgs[:] = 255
        plan = fht.Plan(w, h, strategy, in_dtype="u8", acc_dtype="i32", quadrants=quads, batch=b)
        assert any(g["u16_pair_D"] for g in plan.describe()["groups"])
        out = plan(torch.from_numpy(imgs).cuda())
        torch.cuda.synchronize()
        for bi in range(b):
            ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
            for k in quads:
                np.testing.assert_array_equal(out[k][bi].cpu().numpy(), ref[k], err_msg=f"{h}x{w} s{strategy} {k}")
