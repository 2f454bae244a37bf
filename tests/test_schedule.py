"""CPU: the host schedule tables (plan.cpp via fht_schedule_json) replayed in
numpy exactly as the kernels execute them are bit-exact vs the oracle."""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht
from tests.schedule_replay import replay, working_cols


def _check(h, w, strategy, bw, S, rng, q=0, lo=-1000, hi=1000, levels=4, tw=32, pass_S=None):
    img = rng.integers(lo, hi, (h, w)).astype(np.int64)
    cols = working_cols(img, q)
    W, H = cols.shape
    sched = fht.schedule(W, H, strategy, bw, levels, tw)
    quads, _ = oracle.fht2d_quadrants(img, strategy)
    expect = quads[oracle.QUADRANTS[q]]  # [s, t]
    for pairs in (False, True):  # one level per step (int64 K2) and level pairs (4-byte K2)
        out = replay(cols, sched, S, pass_S, pairs=pairs)
        np.testing.assert_array_equal(out.T, expect, err_msg=f"pairs={pairs}")
    assert sched["additions"] == oracle.count_additions_tree(W, H, strategy)


@pytest.mark.parametrize("strategy", [0, 1])
@pytest.mark.parametrize("bw,levels,tw", [(1, 1, 1), (2, 2, 3), (4, 4, 32), (8, 3, 5), (32, 4, 32), (4, 8, 2)])
def test_all_small_sizes(strategy, bw, levels, tw):
    rng = np.random.default_rng(bw * 10 + strategy)
    for w in range(1, 41):
        for h in (1, 2, 3, 7, 16, 33):
            _check(h, w, strategy, bw, S=8, rng=rng, levels=levels, tw=tw, pass_S=5)


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_quadrant_maps_nonsquare(q):
    rng = np.random.default_rng(q)
    for (h, w) in [(23, 37), (37, 23), (5, 64), (64, 5)]:
        for strategy in (0, 1):
            _check(h, w, strategy, 8, S=16, rng=rng, q=q)


@pytest.mark.parametrize("n", [509, 1000, 1024])
@pytest.mark.parametrize("strategy", [0, 1])
def test_config_widths(n, strategy):
    rng = np.random.default_rng(n)
    _check(9, n, strategy, 32, S=4, rng=rng, lo=0, hi=256, pass_S=4)
    _check(23, n, strategy, 32, S=8, rng=rng, lo=0, hi=256, levels=2, tw=7, pass_S=16)


def test_tweaked_block_structure():
    # every maximal <=32 subtree is an aligned 32-block but one.
    for n, rem in [(1000, 8), (3001, 25), (8191, 31), (509, 29)]:
        s = fht.schedule(n, 1, 1, 32)
        widths = [s["shapes"][b[1]]["width"] for b in s["blocks"]]
        assert sorted(set(widths)) == sorted({32, rem})
        assert widths.count(rem) == 1
        assert all(b[0] % 32 == 0 for b in s["blocks"] if s["shapes"][b[1]]["width"] == 32)
        # the depth of the tree is ceil(log2 n): 5 block levels + the fused passes
        depth = max(b[2] + s["shapes"][b[1]]["steps"] for b in s["blocks"])
        assert depth == int(np.ceil(np.log2(n)))
        assert sum(p["levels"] for p in s["passes"]) == depth - 5


def test_halo_never_exceeds_block_width():
    for strategy in (0, 1):
        for wb in range(1, 65):
            s = fht.schedule(wb, 3, strategy, 64, 4, 32)
            assert s["root_is_block"] == 1
            assert s["shapes"][0]["halo"] <= wb - 1
