"""Latency of the reference-style entry points (host int64 image in, host int64
Hough image out) against the compiled reference on one host thread."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
from paper_2411_07351_b200 import fht
import oracle
rng = np.random.default_rng(0)
for n in (509, 1024, 3001):
    img = rng.integers(0, 256, (n, n)).astype(np.int64)
    fht.fht2d_counted(img, "tweaked")
    t = time.perf_counter(); k = 20
    for _ in range(k): r = fht.fht2d_counted(img, "tweaked")
    dt = (time.perf_counter() - t) / k
    t = time.perf_counter(); kk = 3 if n < 3000 else 1
    for _ in range(kk): ref = oracle.ref_fht2d_counted(img, 1) if hasattr(oracle, "ref_fht2d_counted") else None
    dr = (time.perf_counter() - t) / kk
    print(n, f"gpu fht2d_counted {dt*1e3:.3f} ms", f"reference (1 thread) {dr*1e3:.1f} ms", ref is not None and np.array_equal(r.hough, ref[0]))
    t = time.perf_counter()
    for _ in range(5): fht.fht2d_quadrants(img, "tweaked")
    print("   quadrants", f"{(time.perf_counter()-t)/5*1e3:.3f} ms")
