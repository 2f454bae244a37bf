"""Golden values for the analysis sweep, computed by the UNMODIFIED reference
(analysis.cpp via oracle/_ref/libfhtref.so): max orthotropic errors
E_S(n), E_T(n) (analysis.cpp:63-91, 156-168) as exact reduced rationals, the
Theorem-2 bound (analysis.cpp:23-28) and separation fractions
(analysis.cpp:231-243).  Run where /root/reference exists:

    make -C oracle && python tests/golden/make_golden_analysis.py
"""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent / "analysis_vectors.npz"
SENTINELS = [1451, 2048, 4095, 4096]


def main():
    lib = oracle.ref()
    i64p = ctypes.POINTER(ctypes.c_int64)
    for f in ("ref_max_orthotropic_error", "ref_separation_fraction", "ref_tweaked_error_bound"):
        getattr(lib, f).restype = ctypes.c_int
    lib.ref_max_orthotropic_error.argtypes = [ctypes.c_int, ctypes.c_int, i64p, i64p, ctypes.c_char_p, ctypes.c_int]
    lib.ref_separation_fraction.argtypes = [ctypes.c_int, ctypes.c_int, i64p, i64p, ctypes.c_char_p, ctypes.c_int]
    lib.ref_tweaked_error_bound.argtypes = [ctypes.c_int, i64p, i64p, ctypes.c_char_p, ctypes.c_int]
    a, b = ctypes.c_int64(), ctypes.c_int64()
    e = ctypes.create_string_buffer(256)
    sizes = list(range(1, 1025)) + SENTINELS
    err = np.zeros((len(sizes), 5), np.int64)  # n, num_S, den_S, num_T, den_T
    for k, n in enumerate(sizes):
        err[k, 0] = n
        for s in (0, 1):
            assert lib.ref_max_orthotropic_error(n, s, ctypes.byref(a), ctypes.byref(b), e, 256) == 0
            err[k, 1 + 2 * s], err[k, 2 + 2 * s] = a.value, b.value
    bound = np.zeros((len(sizes), 3), np.int64)
    for k, n in enumerate(sizes):
        assert lib.ref_tweaked_error_bound(n, ctypes.byref(a), ctypes.byref(b), e, 256) == 0
        bound[k] = (n, a.value, b.value)
    sep = []
    for n_max in (64, 512, 1024, 4096):
        t = time.time()
        assert lib.ref_separation_fraction(n_max, 8, ctypes.byref(a), ctypes.byref(b), e, 256) == 0
        sep.append((n_max, a.value, b.value))
        print(f"separation_fraction({n_max}) = {a.value}/{b.value} ({time.time() - t:.1f} s)")
    np.savez_compressed(OUT, errors=err, bound=bound, separation=np.array(sep, np.int64))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
