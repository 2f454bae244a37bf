"""Where the reference-style fht2d_quadrants call spends its time at 3001^2:
fresh (never touched) output pages, touched pageable pages, pinned pages."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_07351_b200._lib import check, lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3001
img = np.random.default_rng(0).integers(0, 256, (n, n)).astype(np.int64)
p = ctypes.POINTER(ctypes.c_int64)
adds = ctypes.c_uint64()


def call(a, outs):
    t = time.perf_counter()
    check(lib().fht_fht2d_quadrants_i64(a.ctypes.data_as(p), n, n, 1, *[o.ctypes.data_as(p) for o in outs],
                                        ctypes.byref(adds)))
    return (time.perf_counter() - t) * 1e3


call(img, [np.empty((n, n), np.int64) for _ in range(4)])
print("fresh pages  ", [round(call(img, [np.empty((n, n), np.int64) for _ in range(4)]), 2) for _ in range(3)])
outs = [np.zeros((n, n), np.int64) for _ in range(4)]
print("touched pages", [round(call(img, outs), 2) for _ in range(3)])
pin = [torch.empty((n, n), dtype=torch.int64).pin_memory().numpy() for _ in range(4)]
pimg = torch.from_numpy(img).pin_memory().numpy()
print("pinned       ", [round(call(pimg, pin), 2) for _ in range(3)])
t = time.perf_counter()
for o in outs:
    o[...] = pin[0]
print("host memcpy of the 4 outputs (1 thread): %.2f ms" % ((time.perf_counter() - t) * 1e3))
t = time.perf_counter()
outs2 = [np.empty((n, n), np.int64) for _ in range(4)]
for o in outs2:
    o.fill(0)
tf = (time.perf_counter() - t) * 1e3
print("fresh pages, touched first: fill %.2f ms + call %.2f ms" % (tf, call(img, outs2)))
