"""Per-GPU step time of c4 at the batch sizes each rank runs under strong
scaling (256 / N images for N = 1, 2, 4, 8): CUDA events, L2 flushed between
steps.  python scripts/batch_sweep.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_07351_b200 import fht, workloads  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
BATCHES = [int(a) for a in sys.argv[1:]] or [256, 128, 64, 32]
ts_256 = None
for n in BATCHES:
    imgs = workloads.make_images("c4", n)
    plan = fht.Plan(509, 509, "tweaked", in_dtype="u8", acc_dtype="i32", batch=n)
    x = torch.from_numpy(imgs).cuda()
    out = plan.alloc_outputs()
    for _ in range(5):
        plan(x, out)
    ts = []
    for _ in range(30):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan(x, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    t = ts[len(ts) // 2]
    eff = f", strong-scaling efficiency at N={256 // n}: {ts_256 / (t * 256 / n):.3f}" if ts_256 and n != 256 else ""
    print(f"images {n:4d}: {t:.4f} ms ({t / n * 256:.4f} ms per 256 images{eff})")
    if n == 256:
        ts_256 = t

# per-kernel times at each batch (events between launches, fht_execute_profiled)
import ctypes  # noqa: E402
from paper_2411_07351_b200._lib import check, lib  # noqa: E402

names = {1: "k1_blocks", 5: "k_stage_u8", 4: "k1p_by32", 2: "k2_pass", 3: "k2_pass_root"}
for n in BATCHES:
    imgs = workloads.make_images("c4", n)
    plan = fht.Plan(509, 509, "tweaked", in_dtype="u8", acc_dtype="i32", batch=n)
    x = torch.from_numpy(imgs).cuda()
    out = plan.alloc_outputs()
    ws = plan.workspace()
    ptrs = (ctypes.c_void_p * 4)(*[out[q].data_ptr() for q in fht.QUADRANTS])
    nl = plan.launches
    ms_arr, kind_arr, b_arr, got = (ctypes.c_float * nl)(), (ctypes.c_int * nl)(), (ctypes.c_double * nl)(), ctypes.c_int()
    res = {}
    for _ in range(5):
        flush.fill_(1)
        check(lib().fht_execute_profiled(plan._h, ctypes.c_void_p(x.data_ptr()), 509 * 509, ptrs, 509 * 509,
                                         ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                         ms_arr, kind_arr, b_arr, nl, ctypes.byref(got)))
        for k, m in zip(list(kind_arr)[:got.value], list(ms_arr)[:got.value]):
            res.setdefault(names[k], []).append(m)
    print(n, {k: round(sorted(v)[len(v) // 2], 4) for k, v in res.items()})
