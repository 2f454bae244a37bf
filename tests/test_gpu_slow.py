"""GPU structure-free oracle (device slow_hough, oracle.cpp:9-25) and the
fast path checked against it bit-exactly at FULL config sizes (where the CPU
Theta(w^2 h) oracle is infeasible)."""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht, workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def test_slow_hough_matches_cpu_oracle_and_golden(golden):
    for row in golden["meta"]:
        i, h, w, strat, adds, qadds = (int(v) for v in row)
        key = f"c{i}_s{strat}_slow"
        if key in golden:
            img = golden[f"c{i}_img"].astype(np.int64)
            np.testing.assert_array_equal(fht.slow_hough(img, strat), golden[key])
    rng = np.random.default_rng(3)
    img = rng.integers(-10_000, 10_000, (29, 47))
    for s in (0, 1):
        np.testing.assert_array_equal(fht.slow_hough(img, s), oracle.slow_hough(img, s))
    with pytest.raises(fht.OverflowBudget):
        fht.slow_hough(np.full((2, 4), 1 << 61, dtype=np.int64))


def _fast(imgs_t, n, quadrants, strategy=1):
    plan = fht.Plan(n, n, strategy, in_dtype="u8", acc_dtype="i32", out_dtype="i64", quadrants=quadrants,
                    batch=imgs_t.shape[0])
    out = plan(imgs_t)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("cfg,quadrants", [("c1", ["vert_pos"]), ("c2", list(fht.QUADRANTS))])
def test_fast_equals_slow_full_size(cfg, quadrants):
    imgs = torch.from_numpy(workloads.make_images(cfg)).cuda()
    n = workloads.CONFIGS[cfg].n
    fast = _fast(imgs, n, quadrants)
    for q in quadrants:
        slow = fht.slow_hough_device(imgs[0], q)
        assert torch.equal(fast[q][0], slow), q


def test_fast_equals_slow_3001_and_c4_sample():
    # c3's size as an integer image (the reference semantics are integer)
    rng = np.random.default_rng(30)
    img = torch.from_numpy(rng.integers(0, 256, (3001, 3001), dtype=np.uint8)).cuda()
    fast = _fast(img[None], 3001, ["horiz_neg", "vert_pos"])
    for q in ("horiz_neg", "vert_pos"):
        assert torch.equal(fast[q][0], fht.slow_hough_device(img, q)), q
    imgs = torch.from_numpy(workloads.make_images("c4", 6)).cuda()
    fast = _fast(imgs, 509, list(fht.QUADRANTS))
    for b in range(6):
        for q in fht.QUADRANTS:
            assert torch.equal(fast[q][b], fht.slow_hough_device(imgs[b], q)), (b, q)


def test_fast_equals_slow_8191_one_quadrant():
    rng = np.random.default_rng(81)
    img = torch.from_numpy(rng.integers(0, 256, (8191, 8191), dtype=np.uint8)).cuda()
    fast = _fast(img[None], 8191, ["vert_neg"])
    assert torch.equal(fast["vert_neg"][0], fht.slow_hough_device(img, "vert_neg"))


def test_simple_strategy_fast_equals_slow_nonsquare():
    rng = np.random.default_rng(7)
    img = torch.from_numpy(rng.integers(0, 256, (777, 1234), dtype=np.uint8)).cuda()
    plan = fht.Plan(1234, 777, "simple", in_dtype="u8", acc_dtype="i32", out_dtype="i64")
    out = plan(img[None])
    for q in fht.QUADRANTS:
        assert torch.equal(out[q][0], fht.slow_hough_device(img, q, "simple")), q
