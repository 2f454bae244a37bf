#!/usr/bin/env python
"""Benchmark of the FHT2D merge DP (arXiv 2411.07351) on B200.

Contract:
  python bench.py --gpus N --steps K --warmup W [--config c4] [--impl ours|reference]

One step = one pass of the hot path over one batch of the workload (default
config c4: 256 binary 509x509 edge maps, all four quadrants, u8 -> int32).
On N GPUs the 256-image batch is sharded 256/N per rank (strong scaling, the
BASELINE.json c4 configuration; --scaling weak gives every rank a whole
batch); no collective on the data path.  `value` is whole-job FHT Gsums/s (BASELINE.json metric:
Q * images * n^2 * ceil(log2 n) nominal adds / s) with inputs resident in HBM;
`e2e` is the same metric through the C-ABI host-buffer call
(fht_execute_host: H2D of the inputs + transform + D2H of every Hough image).
Between timed steps L2 is flushed (a 512 MiB write, untimed); each step is
timed with CUDA events on the launching stream; the max over ranks is taken.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2411_07351_b200 import fht, shard, workloads  # noqa: E402
from paper_2411_07351_b200._lib import check, lib  # noqa: E402

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="tweaked", choices=["simple", "tweaked"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay one captured CUDA graph per step instead of launching through the API "
                         "(measured: no gain; programmatic dependent launch already hides the gaps)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-weak", action="store_true", help="skip the extra weak-scaling measurement at N > 1")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="batch configs on N GPUs: strong = BASELINE's one batch sharded 1/N per GPU "
                         "(images/s = batch / max t); weak = a whole batch per GPU")
    return ap.parse_args()


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    import platform

    return platform.processor() or "unknown"


def hbm_peak():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, window=None):
        """Summarise the samples taken inside `window` = (t0, t1) wall-clock
        (the timed region); all samples if fewer than 2 fall inside."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        scope = "all samples"
        if window is not None:
            inside = [(t, ln) for t, ln in lines if window[0] - 0.05 <= t <= window[1] + 0.05]
            if len(inside) >= 2:
                lines, scope = inside, "timed region"
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "scope": scope}


# ---------------------------------------------------------------- CPU arm
def cpu_baseline(cfg: str, strategy: int, seconds: float, threads: int | None = None):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference library, fht::fht2d_quadrants / fht2d_counted) on this host,
    images across `threads` host threads, on a bounded sample of the workload.
    Falls back to the C restatement (oracle/liboracle.so) if _ref is absent."""
    import oracle

    c = workloads.CONFIGS[cfg]
    threads = threads or oracle.host_threads()
    kind = "reference" if oracle.ref_available() else "port"
    quads = c.quadrants
    mask = sum(1 << workloads.ALL_Q.index(q) for q in quads)
    # Enough images per call that the (image, quadrant) items cover every host
    # thread (independent steps run side by side for batch-1 configs), capped
    # by host memory: the reference holds ~4 int64 planes per item in flight.
    per = max(min(threads, c.batch), -(-threads // len(quads)))
    try:
        import psutil
        fit_items = max(1, int(0.5 * psutil.virtual_memory().available) // (32 * c.n * c.n))
        threads = min(threads, fit_items)
        per = max(1, min(per, -(-fit_items // len(quads))))
    except ImportError:  # pragma: no cover
        pass
    if c.dtype == "u8":
        imgs = workloads.make_images(cfg, per)
        proxy = ""
    else:
        # The reference has no float path: time its int64 path on
        # same-size integer images ("int64 proxy": same add tree, 8-byte cells).
        imgs = np.random.default_rng(0).integers(0, 256, (per, c.n, c.n), dtype=np.uint8)
        proxy = " (int64 proxy: reference has no float path)"
    fn = oracle.ref_batch_quadrants_u8 if kind == "reference" else oracle.batch_quadrants_u8_port
    t0 = time.perf_counter()
    done = 0
    while True:
        fn(imgs, strategy, threads=threads, mask=mask)
        done += per
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    sums = len(quads) * done * c.n * c.n * int(np.ceil(np.log2(c.n)))
    # work items (oracle/ref_shim.cpp ref_batch_quadrants_u8): whole images through the
    # reference's fht2d_quadrants when there are at least as many images as threads,
    # else (image, quadrant) pairs
    per_image = mask == 15 and per >= threads
    used = min(threads, per if per_image else per * len(quads))
    items = "images (fht::fht2d_quadrants each)" if per_image else "(image, quadrant) items"
    return {"value": sums / dt / 1e9, "unit": "Gsums/s", "cores": used, "kind": kind, "cpu_model": cpu_model(),
            "sample": f"{done} image(s) of {cfg} ({c.n}x{c.n}, {len(quads)} quadrant(s)){proxy}, "
                      f"{dt:.2f} s, {items} over {used} host thread(s)"}


def cpu_single_thread(cfg: str, strategy: int, seconds: float):
    """The reference as it runs: one host thread, fht2d_quadrants (or fht2d for
    a one-quadrant config) image after image (quadrants.cpp:23-41,
    transform.cpp:62-85).  Large images: whole (image, quadrant) transforms
    until `seconds` have passed (at least one), counted per quadrant."""
    import oracle

    c = workloads.CONFIGS[cfg]
    kind = "reference" if oracle.ref_available() else "port"
    fn = oracle.ref_batch_quadrants_u8 if kind == "reference" else oracle.batch_quadrants_u8_port
    if c.dtype == "u8":
        img = workloads.make_images(cfg, 1)
        proxy = ""
    else:
        img = np.random.default_rng(0).integers(0, 256, (1, c.n, c.n), dtype=np.uint8)
        proxy = " (int64 proxy: reference has no float path)"
    # one quadrant per call keeps a sample of the largest image bounded; every
    # quadrant of a square image costs the same
    full = sum(1 << workloads.ALL_Q.index(q) for q in c.quadrants)
    mask = full if c.n * c.n * len(c.quadrants) <= (4 << 20) else 1 << workloads.ALL_Q.index(c.quadrants[0])
    nq = bin(mask).count("1")
    t0 = time.perf_counter()
    calls = 0
    while True:
        fn(img, strategy, threads=1, mask=mask)
        calls += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    sums = nq * calls * c.n * c.n * int(np.ceil(np.log2(c.n)))
    return {"value": sums / dt / 1e9, "unit": "Gsums/s", "cores": 1, "kind": kind,
            "sample": f"{calls} x {nq} quadrant(s) of one {c.n}x{c.n} image of {cfg}{proxy}, {dt:.2f} s, 1 thread"}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import oracle

    c = workloads.CONFIGS[args.config]
    strategy = 0 if args.strategy == "simple" else 1
    threads = oracle.host_threads()
    # each step: whole rounds of one image per host thread for at least
    # 0.5 s (a 0.04 s step was too short for a stable median)
    for _ in range(args.warmup):
        cpu_baseline(args.config, strategy, 0.0, threads)
    per_step = []
    vals = []
    for _ in range(args.steps):
        r = cpu_baseline(args.config, strategy, 0.5, threads)
        vals.append(r["value"])
        per_step.append(r)
    value = statistics.median(vals)
    sample = per_step[-1]
    line = {
        "impl": "reference", "metric": "FHT Gsums/s", "value": value, "unit": "Gsums/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": args.scaling if c.batch > 1 else "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.config, "description": c.description, "strategy": args.strategy},
        "cpu_baseline": {"value": value, "unit": "Gsums/s", "cores": sample["cores"], "kind": sample["kind"],
                         "cpu_model": sample.get("cpu_model"),
                         "sample": sample["sample"]},
        "e2e": {"value": value, "unit": "Gsums/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
ESZ = {"u8": 1, "i32": 4, "i64": 8, "f32": 4}


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)  # before the process group: NCCL binds this rank to its GPU
    dev = torch.device("cuda", local)
    if ws > 1:
        # NCCL across GPUs; FHT_DIST_BACKEND=gloo lets several ranks share one
        # GPU for functional testing (their kernels never wait on each other).
        # More local ranks than GPUs (a functional run on one box) cannot use
        # NCCL (one rank per device): fall back to gloo for the few host-side
        # collectives (barrier, timing max); nothing on the data path changes.
        shared_gpu = int(os.environ.get("LOCAL_WORLD_SIZE", ws)) > torch.cuda.device_count()
        backend = os.environ.get("FHT_DIST_BACKEND", "gloo" if shared_gpu else "nccl")
        kw = {"device_id": dev} if backend == "nccl" else {}
        dist.init_process_group(backend, init_method="env://", **kw)
    c = workloads.CONFIGS[args.config]
    strategy = 0 if args.strategy == "simple" else 1

    root_split = None
    n_local = c.batch  # images this rank transforms per step
    if c.batch == 1 and ws > 1:
        # one large image: its quadrants over the ranks; with more ranks than
        # quadrants, pairs of ranks split a quadrant's root (each computes one
        # child subtree, the exchange fused into its last pass, each merges
        # half the root) -- every quadrant owned (shard.image_assignment)
        a = shard.image_assignment(ws, rank, c.quadrants)
        my_q = list(a.quadrants)
        root_split = (a.side, a.peer) if a.side is not None else None
        imgs = workloads.make_images(args.config, 1)
        scaling = "strong"
        sums_per_step = workloads.nominal_sums(args.config)
    elif ws > 1 and args.scaling == "strong":
        # BASELINE's batch sharded across the GPUs: 256 / N images per rank,
        # images/s = 256 / (max over ranks of the step time); no collective
        sh = shard.batch_shard(c.batch, ws, rank)
        n_local = sh.count
        my_q = list(c.quadrants) if n_local > 0 else []
        imgs = workloads.make_images(args.config, max(1, n_local), offset=sh.start)
        scaling = "strong"
        sums_per_step = workloads.nominal_sums(args.config)
    else:
        # a whole batch per rank, no collective on the data path (weak scaling;
        # at N = 1 both readings are the same workload: report the requested one)
        my_q = list(c.quadrants)
        imgs = workloads.make_images(args.config, c.batch, offset=rank * c.batch)
        scaling = "weak" if ws > 1 else (args.scaling if c.batch > 1 else "strong")
        sums_per_step = workloads.nominal_sums(args.config) * ws
    if not my_q:  # more ranks than work: this rank idles but joins the timing
        my_q = None
    plan = fht.Plan(c.n, c.n, strategy, in_dtype=c.dtype, acc_dtype=c.acc, quadrants=my_q or [c.quadrants[0]],
                    batch=max(1, n_local), device=local)
    x = torch.from_numpy(imgs).to(dev)
    out = plan.alloc_outputs()
    wsbuf = plan.workspace()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    cells = c.n * c.n

    ptrs = (ctypes.c_void_p * 4)()
    for i, q in enumerate(fht.QUADRANTS):
        ptrs[i] = out[q].data_ptr() if q in out else None

    if root_split is not None:
        rs_backend = shard.GpuRootBackend(strategy, c.dtype, c.acc)

    graph = None

    def step():
        if my_q is None:
            return
        if graph is not None:
            graph.replay()
            return
        if root_split is not None:
            shard.root_split_quadrant(x[0], my_q[0], strategy, side=root_split[0], backend=rs_backend,
                                      peer=root_split[1])
            return
        check(lib().fht_execute(plan._h, ctypes.c_void_p(x.data_ptr()), cells, ptrs, cells,
                                ctypes.c_void_p(wsbuf.data_ptr() if wsbuf is not None else 0),
                                ctypes.c_void_p(stream.cuda_stream)))

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    if args.graph and my_q is not None and root_split is None:
        # one execute (all its launches, the auxiliary-stream fork/join and the
        # programmatic launch edges) captured once and replayed per step
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            check(lib().fht_execute(plan._h, ctypes.c_void_p(x.data_ptr()), cells, ptrs, cells,
                                    ctypes.c_void_p(wsbuf.data_ptr() if wsbuf is not None else 0),
                                    ctypes.c_void_p(cap.cuda_stream)))
        torch.cuda.synchronize()
        graph = g
        for _ in range(args.warmup):
            flush.fill_(1)
            step()
        torch.cuda.synchronize()
    t_soak = time.perf_counter()
    while True:  # untimed soak: clocks settle under load
        for _ in range(8):
            flush.fill_(1)
            step()
        torch.cuda.synchronize()
        go = time.perf_counter() - t_soak < 1.5  # a fresh box's clocks take a moment to ramp
        if ws > 1:  # every rank runs the same number of steps (the root split's steps are collective)
            flag = torch.tensor([1 if go else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            go = bool(flag.item())
        if not go:
            break
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_wall0 = time.time()
    for s, e in evs:
        flush.fill_(1)  # L2 flush, outside the timed interval
        s.record(stream)
        step()
        e.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    clocks = sampler.stop((t_wall0, t_wall1))
    total_ms = sum(s.elapsed_time(e) for s, e in evs)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = sums_per_step / (ms_per_step * 1e-3) / 1e9

    # Per-kernel live timing (events between launches, same stream) for the roofline.
    nl = plan.launches
    ms_arr = (ctypes.c_float * nl)()
    kind_arr = (ctypes.c_int * nl)()
    bytes_arr = (ctypes.c_double * nl)()
    got = ctypes.c_int()
    per_launch = []
    for _ in range(3):
        flush.fill_(1)
        check(lib().fht_execute_profiled(plan._h, ctypes.c_void_p(x.data_ptr()), cells, ptrs, cells,
                                         ctypes.c_void_p(wsbuf.data_ptr() if wsbuf is not None else 0),
                                         ctypes.c_void_p(stream.cuda_stream), ms_arr, kind_arr, bytes_arr, nl,
                                         ctypes.byref(got)))
        per_launch.append(list(ms_arr)[:got.value])
    kinds = list(kind_arr)[:got.value]
    launch_bytes = list(bytes_arr)[:got.value]
    med = [statistics.median(v) for v in zip(*per_launch)]
    by_kind: dict[int, list] = {}
    for kd, ms, b in zip(kinds, med, launch_bytes):
        by_kind.setdefault(kd, []).append((ms, b))
    names = {1: "k1_blocks", 5: "k_stage_u8", 4: "k1p_by32", 2: "k2_pass", 3: "k2_pass_root"}
    kernel_share = {names[kd]: sum(m for m, _ in v) for kd, v in by_kind.items()}
    dom = max(by_kind, key=lambda kd: sum(m for m, _ in by_kind[kd]))
    dom_ms = statistics.mean(m for m, _ in by_kind[dom])
    dom_bytes = statistics.mean(b for _, b in by_kind[dom])
    peak, peak_src = hbm_peak()
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    # the step's algorithmic bytes exclude the u8 staging copies (kind 5): they
    # are this design's overhead traffic, reported on their own
    total_bytes = sum(b for kd, b in zip(kinds, launch_bytes) if kd != 5)
    staging_bytes = sum(b for kd, b in zip(kinds, launch_bytes) if kd == 5)
    step_gbs = total_bytes / (ms_per_step * 1e-3) / 1e9  # over the event-timed step, not the serialised launches
    roofline = {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                "algorithmic_bytes_per_launch": int(dom_bytes), "avg_launch_ms": round(dom_ms, 5),
                "step_algorithmic_bytes": int(total_bytes), "staging_bytes": int(staging_bytes),
                "step_gbs": round(step_gbs, 1),
                "kernel_ms": {k2: round(v, 4) for k2, v in kernel_share.items()},
                "kernel_gbs": {names[kd]: round(sum(b for _, b in v) / (sum(m for m, _ in v) * 1e-3) / 1e9, 1)
                               for kd, v in by_kind.items()}}
    # The north star's per-level design (one HBM pass per tree level) is HBM-
    # bound; its floor at 100 % of the measured bandwidth is
    # Q * imgs * n^2 * (e_in + e_acc + 2 e_acc (levels - 1)) / peak (SURVEY §8d,
    # K = ceil(log2 n) passes).  The fused passes here are shared-memory bound
    # (low per-pass HBM fraction) yet beat that floor by this factor.
    levels = int(np.ceil(np.log2(c.n)))
    imgs_here = n_local
    nq_here = len(my_q) if my_q else 0
    unfused = nq_here * imgs_here * c.n * c.n * (ESZ[c.dtype] + ESZ[c.acc] + 2 * ESZ[c.acc] * (levels - 1))
    floor_ms = unfused / (peak * 1e9) * 1e3
    roofline["unfused_hbm_floor_ms"] = round(floor_ms, 4)
    roofline["vs_unfused_floor"] = round(floor_ms / ms_per_step, 3) if ms_per_step > 0 else None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            tr = pj.get(args.config, {}).get(names[dom])
            if tr:
                roofline["traffic"] = tr
                # ncu cannot run inside the timed bench: the DRAM bytes (and the
                # LSU / issue fractions below) come from one --set full capture of
                # this build, regenerated with every kernel change
                roofline["traffic_source"] = "profiles/ncu_traffic.json (ncu --set full, same build)"
            # what actually binds the kernel (ncu, same capture): LSU/shared
            # data-pipe wavefronts and issue slots, as fractions of peak
            lsu = pj.get("lsu_issue", {}).get(args.config, {}).get(names[dom])
            if lsu:
                roofline["lsu_pipe_frac_ncu"], roofline["issue_frac_ncu"] = lsu
                # the kernel's floor if its LSU data pipe (shared-memory and
                # global wavefronts, one per SM clock) ran at 100 %, and the
                # HBM fraction that floor would give: why frac < 1
                roofline["lsu_floor_ms"] = round(lsu[0] * dom_ms, 4)
                roofline["frac_at_lsu_floor"] = round(achieved / lsu[0] / peak, 4)
        except Exception:
            pass

    # e2e through the C-ABI host-buffer call (pinned host memory).
    e2e = None
    if not args.no_e2e and my_q is not None and root_split is None:
        h_in = torch.from_numpy(imgs).pin_memory()
        h_out = {q: torch.empty(out[q].shape, dtype=out[q].dtype).pin_memory() for q in out}
        optrs = [h_out[q].data_ptr() if q in h_out else None for q in fht.QUADRANTS]
        st = torch.cuda.Stream(dev)
        for _ in range(2):
            plan.execute_host_ptrs(h_in.data_ptr(), optrs, st.cuda_stream)
        n_e2e = max(3, min(args.steps, 10))
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            plan.execute_host_ptrs(h_in.data_ptr(), optrs, st.cuda_stream)  # synchronises its stream
        e2e_s = torch.tensor([(time.perf_counter() - t0) / n_e2e], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_s.item())
        e2e = {"value": sums_per_step / e2e_s / 1e9, "unit": "Gsums/s",
               "h2d_bytes_per_step": int(h_in.numel() * h_in.element_size()),
               "d2h_bytes_per_step": int(sum(v.numel() * v.element_size() for v in h_out.values())),
               "ms_per_step": round(e2e_s * 1e3, 3), "call": "fht_execute_host (C ABI, pinned host buffers)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, strategy, args.cpu_seconds)
        cpu["single_thread"] = cpu_single_thread(args.config, strategy, max(1.0, args.cpu_seconds / 2))

    weak = None
    if ws > 1 and scaling == "strong" and c.batch > 1 and my_q is not None and not args.no_weak:
        # extra key: the weak-scaling figure (a whole batch per GPU) beside the
        # strong-scaling headline
        wplan = fht.Plan(c.n, c.n, strategy, in_dtype=c.dtype, acc_dtype=c.acc, quadrants=my_q, batch=c.batch,
                         device=local)
        wx = torch.from_numpy(workloads.make_images(args.config, c.batch, offset=rank * c.batch)).to(dev)
        wout = wplan.alloc_outputs()
        for _ in range(2):
            wplan(wx, out=wout)
        nw = max(3, min(args.steps, 10))
        torch.cuda.synchronize()
        dist.barrier()
        ws_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nw)]
        for s0, e0 in ws_ev:
            flush.fill_(1)
            s0.record(stream)
            wplan(wx, out=wout)
            e0.record(stream)
        torch.cuda.synchronize()
        wt = torch.tensor([sum(a.elapsed_time(b) for a, b in ws_ev) / nw], dtype=torch.float64, device=dev)
        dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        wms = float(wt.item())
        weak = {"value": round(workloads.nominal_sums(args.config) * ws / (wms * 1e-3) / 1e9, 3),
                "unit": "Gsums/s", "ms_per_step": round(wms, 4), "images_per_s": round(c.batch * ws / (wms * 1e-3), 1),
                "images_per_gpu": c.batch}
        del wplan, wx, wout

    if rank == 0:
        line = {
            "metric": "FHT Gsums/s", "value": round(value, 3), "unit": "Gsums/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": c.acc,
            "data": "synthetic (seeded, BASELINE.json config shapes/distributions)",
            "config": {"workload": args.config, "description": c.description, "n": c.n,
                       "images_per_gpu": n_local, "quadrants": len(c.quadrants), "strategy": args.strategy,
                       "cuda_graph": graph is not None,
                       "in_dtype": c.dtype, "acc_dtype": c.acc,
                       "parallelism": (f"batch-shard x{ws} ({c.batch}/{ws} images per GPU)" if c.batch > 1 and scaling == "strong"
                                       else f"batch per GPU x{ws}" if c.batch > 1
                                       else "root-split x2 per quadrant" if ws >= 2 * len(c.quadrants)
                                       else f"root-split x2 for {ws - len(c.quadrants)} of {len(c.quadrants)} quadrants"
                                       if ws > len(c.quadrants)
                                       else f"quadrant-split x{ws}"),
                       "l2": "flushed between timed steps (512 MiB write, untimed)"},
            "images_per_s": round((c.batch * ws if scaling == "weak" else c.batch) / (ms_per_step * 1e-3), 1),
            "weak_scaling": weak,
            "hbm_gbs_step": round(step_gbs, 1),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": plan.launches * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
