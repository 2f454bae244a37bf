"""Pin the CPU oracle (oracle/fht_oracle.c) before trusting it.

* against the golden vectors the UNMODIFIED reference produced
  (tests/golden/make_golden.py -> reference_vectors.npz);
* against the SPEC.md known-answer examples;
* against the compiled reference itself (oracle/_ref) when it is present.
"""
import numpy as np
import pytest

import oracle

S, T = oracle.SIMPLE, oracle.TWEAKED


def _cases(golden):
    for row in golden["meta"]:
        i, h, w, strat, adds, qadds = (int(v) for v in row)
        yield i, h, w, strat, adds, qadds


def test_golden_fht2d_and_counts(golden):
    n = 0
    for i, h, w, strat, adds, qadds in _cases(golden):
        img = golden[f"c{i}_img"].astype(np.int64)
        j, a = oracle.fht2d_counted_i64(img, strat)
        assert a == adds
        np.testing.assert_array_equal(j, golden[f"c{i}_s{strat}_fht2d"])
        n += 1
    assert n == 32


@pytest.mark.parametrize("dtype", [np.int64, np.int32, np.float64])
def test_golden_quadrants_all_dtypes(golden, dtype):
    for i, h, w, strat, adds, qadds in _cases(golden):
        img = golden[f"c{i}_img"].astype(dtype)
        q, a = oracle.fht2d_quadrants(img, strat, dtype=dtype)
        assert a == qadds
        for k in oracle.QUADRANTS:
            np.testing.assert_array_equal(q[k], golden[f"c{i}_s{strat}_{k}"].astype(dtype))


def test_golden_slow_hough(golden):
    seen = 0
    for i, h, w, strat, adds, qadds in _cases(golden):
        key = f"c{i}_s{strat}_slow"
        if key in golden:
            img = golden[f"c{i}_img"].astype(np.int64)
            np.testing.assert_array_equal(oracle.slow_hough(img, strat), golden[key])
            seen += 1
    assert seen >= 20


def test_golden_patterns(golden):
    for row in golden["patterns"]:
        strat, n, t = (int(v) for v in row[:3])
        assert oracle.pattern(n, t, strat) == [int(v) for v in row[3:3 + n]]


def test_golden_counts(golden):
    for strat, w, h, c in golden["counts"]:
        assert oracle.count_additions_tree(int(w), int(h), int(strat)) == int(c)


# ---- SPEC.md known answers
def test_spec_splits_and_rounding():
    assert oracle.split_width(2, S) == (1, 1)
    assert oracle.split_width(5, S) == (2, 3)
    assert oracle.split_width(17, S) == (8, 9)
    assert oracle.split_width(2, T) == (1, 1)
    assert oracle.split_width(17, T) == (16, 1)
    assert oracle.split_width(6, T) == (4, 2)
    assert oracle.round_half_up_ratio(1, 3) == 0
    assert oracle.round_half_up_ratio(2, 3) == 1
    assert oracle.round_half_up_ratio(1, 2) == 1


def test_spec_2x2_example():
    a, b, c, d = 3, 5, 7, 11
    img = np.array([[a, b], [c, d]], dtype=np.int64)  # I(0,0)=a I(1,0)=b I(0,1)=c I(1,1)=d
    j, _ = oracle.fht2d_counted_i64(img, T)
    # J(t, s) stored as j[s, t]
    assert j[0, 0] == a + b and j[1, 0] == c + d and j[0, 1] == a + d and j[1, 1] == c + b


def test_spec_counts_and_patterns():
    assert oracle.count_additions_tree(1, 7, T) == 0
    assert oracle.count_additions_tree(3, 3, S) == 15
    assert oracle.count_additions_tree(17, 17, T) == 1377
    assert oracle.pattern(1, 0, T) == [0]
    assert oracle.pattern(4, 3, T) == [0, 1, 2, 3]
    assert oracle.pattern(3, 2, T) == [0, 1, 2]
    assert oracle.pattern(4, 1, T) == [0, 0, 1, 1]
    assert [oracle.pattern(4, t, T) for t in range(4)] == [[0, 0, 0, 0], [0, 0, 1, 1], [0, 1, 1, 2], [0, 1, 2, 3]]
    assert [oracle.pattern(2, t, S) for t in range(2)] == [[0, 0], [0, 1]]


def test_spec_properties_small():
    rng = np.random.default_rng(1)
    for n in (1, 2, 4, 8, 16, 32, 64):  # power-of-two coincidence
        img = rng.integers(0, 256, (n, n))
        np.testing.assert_array_equal(oracle.fht2d_counted_i64(img, S)[0], oracle.fht2d_counted_i64(img, T)[0])
    img = rng.integers(-50, 50, (13, 21))
    j = oracle.fht2d_counted_i64(img, T)[0]
    assert (j.sum(axis=0) == img.sum()).all()  # mass conservation
    r = 5  # shift equivariance
    js = oracle.fht2d_counted_i64(np.roll(img, -r, axis=0), T)[0]
    np.testing.assert_array_equal(js, np.roll(j, -r, axis=0))
    img2 = rng.integers(-50, 50, (13, 21))  # linearity
    j2 = oracle.fht2d_counted_i64(img2, T)[0]
    np.testing.assert_array_equal(oracle.fht2d_counted_i64(3 * img - 2 * img2, T)[0], 3 * j - 2 * j2)


def test_overflow_and_empty():
    with pytest.raises(oracle.OverflowBudget):
        oracle.fht2d_counted_i64(np.full((2, 4), 1 << 61, dtype=np.int64), T)
    with pytest.raises(oracle.InvalidArgument):
        oracle.fht2d_counted_i64(np.zeros((0, 3), dtype=np.int64), T)


def test_fp32_restatement_close_to_fp64():
    rng = np.random.default_rng(7)
    img = rng.standard_normal((101, 97)).astype(np.float32)
    j32, _ = oracle.fht2d(img, T, dtype=np.float32)
    j64, _ = oracle.fht2d(img.astype(np.float64), T, dtype=np.float64)
    l1, _ = oracle.fht2d(np.abs(img).astype(np.float64), T, dtype=np.float64)
    assert (np.abs(j32 - j64) <= 1e-5 * l1).all()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_port_matches_compiled_reference():
    rng = np.random.default_rng(3)
    for (h, w) in [(1, 1), (5, 1), (1, 5), (24, 24), (33, 47), (47, 33), (3, 100), (100, 3), (64, 65)]:
        for strat in (S, T):
            img = rng.integers(-10_000, 10_000, (h, w))
            jr, ar = oracle.ref_fht2d_counted(img, strat)
            jp, ap = oracle.fht2d_counted_i64(img, strat)
            np.testing.assert_array_equal(jr, jp)
            assert ar == ap
            qr, tr = oracle.ref_fht2d_quadrants(img, strat)
            qp, tp = oracle.fht2d_quadrants(img, strat)
            assert tr == tp
            for k in oracle.QUADRANTS:
                np.testing.assert_array_equal(qr[k], qp[k])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_batch_baseline_helpers_agree():
    rng = np.random.default_rng(4)
    imgs = rng.integers(0, 256, (3, 29, 31), dtype=np.uint8)
    a = oracle.ref_batch_quadrants_u8(imgs, T, threads=2, want_output=True)
    b = oracle.batch_quadrants_u8_port(imgs, T, threads=2, want_output=True)
    np.testing.assert_array_equal(a, b)
    q, _ = oracle.ref_fht2d_quadrants(imgs[1].astype(np.int64), T)
    np.testing.assert_array_equal(a[1, 2], q["vert_pos"].ravel())


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_port_matches_compiled_reference_every_small_shape():
    """Every w, h <= 20, both strategies, all four quadrants and the addition
    counts, against the reference library compiled from its own sources
    (transform.cpp:62-85, quadrants.cpp:23-41)."""
    rng = np.random.default_rng(5)
    for h in range(1, 21):
        for w in range(1, 21):
            img = rng.integers(-1000, 1000, (h, w))
            for strat in (S, T):
                qr, tr = oracle.ref_fht2d_quadrants(img, strat)
                qp, tp = oracle.fht2d_quadrants(img, strat)
                assert tr == tp, (h, w, strat)
                for k in oracle.QUADRANTS:
                    np.testing.assert_array_equal(qr[k], qp[k], err_msg=f"{h}x{w} {k} strategy {strat}")


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_port_matches_compiled_reference_random_shapes():
    """Seeded random shapes up to 300 wide (non-powers of two, thin images)."""
    rng = np.random.default_rng(6)
    for _ in range(12):
        h, w = (int(v) for v in rng.integers(1, 301, 2))
        strat = int(rng.integers(0, 2))
        img = rng.integers(0, 256, (h, w))
        jr, ar = oracle.ref_fht2d_counted(img, strat)
        jp, ap = oracle.fht2d_counted_i64(img, strat)
        np.testing.assert_array_equal(jr, jp, err_msg=f"{h}x{w} strategy {strat}")
        assert ar == ap
