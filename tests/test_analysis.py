"""Analysis sweep (analysis.cpp) vs golden values the reference computed
(tests/golden/make_golden_analysis.py): exact E_S(n), E_T(n) for n <= 1024
and the sentinels, the Theorem-2 bound, and separation fractions up to 4096
(the paper's §5 claims)."""
from fractions import Fraction

import numpy as np
import pytest

from paper_2411_07351_b200 import analysis


@pytest.fixture(scope="module")
def gold():
    from pathlib import Path

    return np.load(Path(__file__).resolve().parent / "golden" / "analysis_vectors.npz")


def test_bounds_and_closed_forms(gold):
    for n, num, den in gold["bound"]:
        assert analysis.tweaked_error_bound(int(n)) == Fraction(int(num), int(den))
    recs = analysis.complexity_series(64)
    for r in recs:
        assert r.f_simple == analysis.closed_form_f_simple(r.n)  # Theorem 1 Eq. (1)
    assert recs[16].f_tweaked == 1377  # f_T(17)
    assert analysis.fast_mode_sizes(5000)[-4:] == [1451, 2048, 4095, 4096]


@pytest.mark.gpu
def test_error_sweep_matches_reference(gold):
    err = gold["errors"]
    sizes = [int(n) for n in err[:, 0]]
    recs = {r.n: r for r in analysis.error_series_for(sizes[:1024])}
    for n, ns, ds, nt, dt in err:
        n = int(n)
        if n in recs:
            assert recs[n].e_simple == Fraction(int(ns), int(ds)), n
            assert recs[n].e_tweaked == Fraction(int(nt), int(dt)), n
    for n, ns, ds, nt, dt in err[1024:]:  # sentinels
        assert analysis.max_orthotropic_error(int(n), "simple") == Fraction(int(ns), int(ds))
        assert analysis.max_orthotropic_error(int(n), "tweaked") == Fraction(int(nt), int(dt))
    ratio = analysis.max_orthotropic_error(1451, "simple") / analysis.max_orthotropic_error(1451, "tweaked")
    assert ratio > Fraction(169, 100)
    assert all(r.e_tweaked <= r.bound for r in recs.values())  # Theorem 2


@pytest.mark.gpu
def test_separation_fraction_matches_reference(gold):
    for n_max, num, den in gold["separation"]:
        assert analysis.separation_fraction(int(n_max)) == Fraction(int(num), int(den))
    assert analysis.separation_fraction(4096) >= Fraction(3638, 10000)  # "no less than 36.38%"
