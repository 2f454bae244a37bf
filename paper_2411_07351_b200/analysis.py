"""The paper's complexity / accuracy analysis (Theorems 1-2, §5 figures),
mirroring the reference's analysis module (analysis.hpp:30-63), with the
Theta(n_max^3) error sweep on the GPU (fht_max_deviation_numerators).

Exact arithmetic throughout: errors and bounds are fractions.Fraction
(the reference's Rational, rational.hpp)."""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from ._lib import check, lib
from .fht import SplitStrategy, _strategy, count_additions_tree


def floor_log2(n: int) -> int:
    if n < 1:
        raise ValueError("floor_log2: argument must be positive")
    return n.bit_length() - 1


def closed_form_f_simple(n: int) -> int:
    """Theorem 1 Eq. (1), analysis.cpp:16-21."""
    if n < 1:
        raise ValueError("closed_form_f_simple: n must be positive")
    q = floor_log2(n)
    return (q + 2) * n * n - (1 << (q + 1)) * n


def tweaked_error_bound(n: int) -> Fraction:
    """Theorem 2 bound floor(log2 n)/6 + 1 - 2^-floor(log2 n), analysis.cpp:23-28."""
    if n < 1:
        raise ValueError("tweaked_error_bound: n must be positive")
    q = floor_log2(n)
    p = 1 << q
    return Fraction(q * p + 6 * p - 6, 6 * p)


def max_deviation_numerators(n_lo: int, n_hi: int, strategy=SplitStrategy.Tweaked) -> np.ndarray:
    """worst[n - n_lo] = max_t,x |x t - pat(n,t)(x) (n-1)| for n in [n_lo, n_hi] (GPU)."""
    out = np.zeros(n_hi - n_lo + 1, dtype=np.int64)
    check(lib().fht_max_deviation_numerators(n_lo, n_hi, _strategy(strategy),
                                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return out


def max_orthotropic_error(n: int, strategy=SplitStrategy.Tweaked) -> Fraction:
    """analysis.hpp:39 (E_S / E_T of Theorem 2), exact."""
    if n < 1:
        raise ValueError("max_orthotropic_error: n must be positive")
    w = int(max_deviation_numerators(n, n, strategy)[0])
    return Fraction(w, n - 1 if n > 1 else 1)


@dataclass
class ComplexityRecord:
    n: int
    f_simple: int
    f_tweaked: int
    norm_simple: float | None
    norm_tweaked: float | None


@dataclass
class ErrorRecord:
    n: int
    e_simple: Fraction
    e_tweaked: Fraction
    bound: Fraction
    norm_simple: float | None
    norm_tweaked: float | None


def complexity_series(n_max: int) -> list[ComplexityRecord]:
    """analysis.cpp:180-198."""
    if n_max < 1:
        raise ValueError("complexity_series: n_max must be positive")
    recs = []
    for n in range(1, n_max + 1):
        fs = count_additions_tree(n, n, SplitStrategy.Simple)
        ft = count_additions_tree(n, n, SplitStrategy.Tweaked)
        d = n * n * math.log2(n) if n > 1 else None
        recs.append(ComplexityRecord(n, fs, ft, fs / d if d else None, ft / d if d else None))
    return recs


def error_series_for(sizes) -> list[ErrorRecord]:
    """analysis.cpp:200-208 for an ascending list of sizes (GPU sweep)."""
    sizes = list(sizes)
    if any(n < 1 for n in sizes) or any(b <= a for a, b in zip(sizes, sizes[1:])):
        raise ValueError("error_series: sizes must be positive and strictly ascending")
    lo, hi = sizes[0], sizes[-1]
    ws = max_deviation_numerators(lo, hi, SplitStrategy.Simple)
    wt = max_deviation_numerators(lo, hi, SplitStrategy.Tweaked)
    recs = []
    for n in sizes:
        den = n - 1 if n > 1 else 1
        es, et = Fraction(int(ws[n - lo]), den), Fraction(int(wt[n - lo]), den)
        sc = 6.0 / math.log2(n) if n > 1 else None
        recs.append(ErrorRecord(n, es, et, tweaked_error_bound(n), float(es) * sc if sc else None,
                                float(et) * sc if sc else None))
    return recs


def error_series(n_max: int) -> list[ErrorRecord]:
    return error_series_for(range(1, n_max + 1))


def fast_mode_sizes(n_max: int) -> list[int]:
    """analysis.cpp:222-229."""
    if n_max < 1:
        raise ValueError("fast_mode_sizes: n_max must be positive")
    return list(range(1, min(n_max, 1024) + 1)) + [s for s in (1451, 2048, 4095, 4096) if s <= n_max]


def separation_fraction(n_max: int) -> Fraction:
    """Fraction of n in [1, n_max] whose Simple error exceeds the Tweaked bound
    (analysis.cpp:231-243)."""
    if n_max < 1:
        raise ValueError("separation_fraction: n_max must be positive")
    ws = max_deviation_numerators(1, n_max, SplitStrategy.Simple)
    count = 0
    for n in range(1, n_max + 1):
        if Fraction(int(ws[n - 1]), n - 1 if n > 1 else 1) > tweaked_error_bound(n):
            count += 1
    return Fraction(count, n_max)
