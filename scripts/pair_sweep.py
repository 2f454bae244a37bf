"""One-off randomized sweep of the u16 pair mode (u8 images, W <= 512, H <= 512,
both strategies, random batches and quadrant masks), bit-exact vs the oracle.
    python scripts/pair_sweep.py [iterations]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2411_07351_b200 import fht  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(2026)
pm = 0
for it in range(iters):
    w = int(rng.integers(65, 513))
    h = int(rng.integers(64, 513))
    strategy = int(rng.integers(2))
    b = int(rng.integers(1, 4))
    mask = int(rng.integers(1, 16))
    quads = [q for i, q in enumerate(oracle.QUADRANTS) if mask & (1 << i)]
    imgs = rng.integers(0, 256, (b, h, w)).astype(np.uint8)
    if rng.random() < 0.2:
        imgs[:] = 255  # the pair mode's 16-bit limit
    plan = fht.Plan(w, h, strategy, in_dtype="u8", acc_dtype="i32", quadrants=quads, batch=b)
    pm += any(g["u16_pair_D"] for g in plan.describe()["groups"])
    out = plan(torch.from_numpy(imgs).cuda())
    torch.cuda.synchronize()
    for bi in range(b):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=np.int32)
        for k in quads:
            if not np.array_equal(out[k][bi].cpu().numpy(), ref[k]):
                print("MISMATCH", it, h, w, strategy, b, k, bi)
                sys.exit(1)
print(f"ok: {iters} plans, {pm} in the pair mode")
