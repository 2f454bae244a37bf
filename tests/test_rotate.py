"""CPU: fht::rotate (transform.cpp:8-14) in the Python mirror against SPEC.md's
examples and the reference's own rotate (oracle/_ref)."""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht


def test_rotate_spec_examples():
    a, b, c, d = 11, 22, 33, 44
    assert list(fht.rotate([a, b, c, d], 0)) == [a, b, c, d]  # identity
    assert list(fht.rotate([a, b, c, d], 1)) == [b, c, d, a]  # u(i) = v((i + r) mod h)
    assert list(fht.rotate([a, b], 1)) == [b, a]  # swap


@pytest.mark.parametrize("h,r", [(1, -1), (1, 1), (4, 4), (4, -1), (0, 0)])
def test_rotate_rejects_shift_outside_range(h, r):
    with pytest.raises(fht.InvalidArgument):
        fht.rotate(np.arange(h), r)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_rotate_matches_reference():
    rng = np.random.default_rng(7)
    for h in (1, 2, 3, 7, 16, 509):
        v = rng.integers(-2**62, 2**62, h, dtype=np.int64)
        for r in sorted({0, min(1, h - 1), h // 2, h - 1}):
            assert np.array_equal(fht.rotate(v, r), oracle.ref_rotate(v, r))
    with pytest.raises(oracle.InvalidArgument):
        oracle.ref_rotate(np.arange(4), 4)


def test_rotate_is_the_merge_shift():
    """The merge reads b[(s + r) mod h] (transform.cpp:53-55): rotate(v, r)[s]."""
    v = np.arange(10, 20, dtype=np.int64)
    for r in range(10):
        assert all(fht.rotate(v, r)[s] == v[(s + r) % 10] for s in range(10))
