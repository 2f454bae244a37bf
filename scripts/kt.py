"""Per-launch kernel times (CUDA events, L2 flushed) for one config, for A/B runs.

    python scripts/kt.py --config c5 [--layout native] [--reps 5]
"""
import argparse
import ctypes
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2411_07351_b200 import fht, workloads  # noqa: E402
from paper_2411_07351_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--layout", default="reference")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
c = workloads.CONFIGS[a.config]
imgs = workloads.make_images(a.config, c.batch)
plan = fht.Plan(c.n, c.n, "tweaked", in_dtype=c.dtype, acc_dtype=c.acc, quadrants=list(c.quadrants), batch=c.batch,
                layout=a.layout)
x = torch.from_numpy(imgs).cuda()
out = plan.alloc_outputs()
ws = plan.workspace()
plan(x, out)
qs = plan.quadrants
ptrs = (ctypes.c_void_p * 4)(*[out[q].data_ptr() if q in out else None for q in ("horiz_pos", "horiz_neg", "vert_pos", "vert_neg")])
cells = c.n * c.n
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
nl = plan.launches
ms_arr = (ctypes.c_float * nl)()
kind_arr = (ctypes.c_int * nl)()
bytes_arr = (ctypes.c_double * nl)()
got = ctypes.c_int()
runs = []
for _ in range(a.reps):
    flush.fill_(1)
    check(lib().fht_execute_profiled(plan._h, ctypes.c_void_p(x.data_ptr()), cells, ptrs, cells,
                                     ctypes.c_void_p(ws.data_ptr() if ws is not None else 0),
                                     ctypes.c_void_p(stream.cuda_stream), ms_arr, kind_arr, bytes_arr, nl,
                                     ctypes.byref(got)))
    runs.append(list(ms_arr)[:got.value])
med = [statistics.median(v) for v in zip(*runs)]
kinds = list(kind_arr)[:got.value]
names = {1: "k1_blocks", 5: "k_stage_u8", 4: "k1p_by32", 2: "k2_pass", 3: "k2_pass_root"}
print(a.config, a.layout, "total %.4f ms" % sum(med),
      " ".join("%s=%.4f" % (names[k], m) for k, m in zip(kinds, med)))
