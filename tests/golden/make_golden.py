"""Generate the golden fixtures in this directory FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

It calls the unmodified reference library (oracle/_ref/libfhtref.so, built
from /root/reference/proj/src by oracle/Makefile) through oracle/ref_shim.cpp:
fht::fht2d_counted (transform.cpp:62), fht::fht2d_quadrants (quadrants.cpp:23),
fht::slow_hough (oracle.cpp:9), fht::fht2d_pattern (pattern.cpp:24) and
fht::count_additions_tree (oracle.cpp:27).  The GPU box has no
/root/reference, so tests read these committed vectors instead.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_vectors.npz"

# (h, w, value_lo, value_hi) -- small, ragged, degenerate and power-of-two shapes
SHAPES = [(1, 1, -5, 5), (7, 1, -50, 50), (1, 7, -50, 50), (2, 2, 0, 10), (3, 3, -9, 9), (4, 5, 0, 256),
          (6, 6, 0, 2), (17, 17, 0, 256), (23, 37, -1000, 1000), (37, 23, -1000, 1000), (47, 33, 0, 256),
          (32, 32, 0, 256), (64, 64, -128, 128), (17, 100, 0, 256), (100, 17, 0, 256), (31, 65, 0, 256)]


def main() -> None:
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref/libfhtref.so missing: run `make -C oracle` where /root/reference exists")
    rng = np.random.default_rng(20241107)
    arrays: dict[str, np.ndarray] = {}
    meta = []
    for i, (h, w, lo, hi) in enumerate(SHAPES):
        img = rng.integers(lo, hi, size=(h, w), dtype=np.int64)
        arrays[f"c{i}_img"] = img.astype(np.int32)
        for strat in (oracle.SIMPLE, oracle.TWEAKED):
            j, adds = oracle.ref_fht2d_counted(img, strat)
            q, qadds = oracle.ref_fht2d_quadrants(img, strat)
            arrays[f"c{i}_s{strat}_fht2d"] = j.astype(np.int32)
            for k, v in q.items():
                arrays[f"c{i}_s{strat}_{k}"] = v.astype(np.int32)
            if w * w * h <= 200_000:
                arrays[f"c{i}_s{strat}_slow"] = oracle.ref_slow_hough(img, strat).astype(np.int32)
            meta.append((i, h, w, strat, adds, qadds))
    arrays["meta"] = np.array(meta, dtype=np.int64)  # case, h, w, strategy, additions, quadrant additions
    # Patterns (Algorithm 2) for every n <= 40, every slope, both strategies.
    pats = []
    for strat in (0, 1):
        for n in range(1, 41):
            for t in range(n):
                v = oracle.ref_pattern(n, t, strat)
                pats.append([strat, n, t] + v + [-1] * (40 - n))
    arrays["patterns"] = np.array(pats, dtype=np.int32)
    # count_additions_tree for w, h <= 40 both strategies (and the config sizes).
    counts = []
    for strat in (0, 1):
        for w in list(range(1, 41)) + [509, 1000, 1024, 1451, 3001, 4096, 8191]:
            for h in (1, 2, 7, 40, w):
                counts.append([strat, w, h, oracle.ref_count_additions_tree(w, h, strat)])
    arrays["counts"] = np.array(counts, dtype=np.int64)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(meta)} transform cases)")


if __name__ == "__main__":
    main()
