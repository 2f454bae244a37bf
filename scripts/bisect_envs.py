"""Run one small u8 plan per environment setting in a subprocess; report ok / crash / mismatch."""
import os
import subprocess
import sys

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_2411_07351_b200 import fht
h, w, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(1)
imgs = rng.integers(0, 256, (b, h, w), dtype=np.uint8)
plan = fht.Plan(w, h, 1, in_dtype="u8", acc_dtype="i32", quadrants="all", batch=b)
d = plan.describe()
out = plan(torch.from_numpy(imgs).cuda()); torch.cuda.synchronize()
ref, _ = oracle.fht2d_quadrants(imgs[0], 1, dtype=np.int32)
bad = [k for k in oracle.QUADRANTS if not np.array_equal(out[k][0].cpu().numpy(), ref[k])]
print("pairD", [g["u16_pair_D"] for g in d["groups"]], "S", [g["S"] for g in d["groups"]], "mismatch" if bad else "ok", bad)
'''

cases = sys.argv[1:] or ["509,509,2"]
envs = ["", "FHT_U16_PAIRS=0", "FHT_U16_PAIRS=0 FHT_K1_STAGE=0", "FHT_U16_PAIRS=0 FHT_K2_PAIRS=0",
        "FHT_U16_PAIRS=0 FHT_K1_OVERLAP=0", "FHT_U16_PAIRS=0 FHT_PDL=0", "FHT_U16_PAIRS=0 FHT_K1_BY32=0",
        "FHT_K1_OVERLAP=0 FHT_PDL=0"]
for case in cases:
    h, w, b = case.split(",")
    for e in envs:
        env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
        for kv in e.split():
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD, h, w, b], env=env, capture_output=True, text=True, timeout=300)
        tail = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else "CRASH " + " | ".join(
            l for l in r.stderr.strip().splitlines()[-3:])
        print(f"{case:12s} {e:45s} {tail}", flush=True)
