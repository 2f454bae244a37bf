"""Device time of one transform per accumulator type (int32 vs int64 vs f32)
on the same image size: the int64 path (values too large for int32 sums,
transform.cpp:16-27's budget) against the int32 one.

    python scripts/bench_acc.py --n 1024 --quadrants 4 --batch 1
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_07351_b200 import fht  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
n, b = a.n, a.batch
sums = 4 * b * n * n * int(np.ceil(np.log2(n)))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for in_dt, acc in (("i32", "i32"), ("i64", "i64"), ("i64", "i64p0"), ("i32", "i64"), ("i32", "i64p0"), ("f32", "f32")):
    p0 = acc == "i64p0"  # int64 plan with pass 0 in int32 (values < 2^20 here: 32 * max|v| < 2^31)
    acc = "i64" if p0 else acc
    tdt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32}[in_dt]
    x = (torch.randint(-(1 << 20), 1 << 20, (b, n, n), dtype=torch.int64) if in_dt != "f32"
         else torch.randn(b, n, n)).to(tdt).cuda()
    plan = fht.Plan(n, n, "tweaked", in_dtype=in_dt, acc_dtype=acc, batch=b, pass0_i32=p0)
    out = plan.alloc_outputs()
    for _ in range(3):
        plan(x, out=out)
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.iters):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        plan(x, out=out)
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    m = float(np.median(ms))
    # per-launch times (events between launches, fht_execute_profiled)
    import ctypes

    from paper_2411_07351_b200._lib import check, lib
    nl = plan.launches
    ms_arr, kind_arr, b_arr, got = (ctypes.c_float * nl)(), (ctypes.c_int * nl)(), (ctypes.c_double * nl)(), ctypes.c_int()
    ptrs = (ctypes.c_void_p * 4)(*[out[q].data_ptr() for q in fht.QUADRANTS])
    ws = plan.workspace()
    check(lib().fht_execute_profiled(plan._h, ctypes.c_void_p(x.data_ptr()), n * n, ptrs, n * n,
                                     ctypes.c_void_p(ws.data_ptr() if ws is not None else 0),
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ms_arr, kind_arr, b_arr,
                                     nl, ctypes.byref(got)))
    names = {1: "K1", 5: "stage", 4: "K1P", 2: "K2", 3: "K2root"}
    per = " ".join(f"{names[kind_arr[i]]}={ms_arr[i]:.3f}" for i in range(got.value))
    print(f"{n}x{n} x{b} in={in_dt} acc={acc}{' (pass 0 int32)' if p0 else ''}: {m:.4f} ms  {sums / m / 1e6:.1f} Gsums/s  [{per}]")
