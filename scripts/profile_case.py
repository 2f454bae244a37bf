"""Run one config's transform a few times (for ncu / compute-sanitizer).

    python scripts/profile_case.py --config c4 --iters 2
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2411_07351_b200 import fht, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--images", type=int, default=None)
ap.add_argument("--strategy", default="tweaked")
a = ap.parse_args()
c = workloads.CONFIGS[a.config]
n_img = a.images or c.batch
imgs = workloads.make_images(a.config, n_img)
plan = fht.Plan(c.n, c.n, a.strategy, in_dtype=c.dtype, acc_dtype=c.acc, quadrants=list(c.quadrants), batch=n_img)
x = torch.from_numpy(imgs).cuda()
out = plan.alloc_outputs()
for _ in range(a.iters):
    plan(x, out)
torch.cuda.synchronize()
print("ok", plan.describe()["launches"], "launches/execute")
