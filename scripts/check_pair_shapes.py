"""Bit-exactness of the pair-mode path on a list of shapes under the current
environment (FHT_* settings), against the oracle; prints one line per shape.

    FHT_TILE_WIDTH=32 FHT_K2_SMEM_KB=125 python scripts/check_pair_shapes.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2411_07351_b200 import fht  # noqa: E402

SHAPES = [(509, 509, 1), (512, 512, 1), (64, 65, 1), (65, 300, 0), (511, 96, 1), (120, 258, 0), (130, 257, 1),
          (333, 77, 0), (257, 511, 1), (300, 65, 0), (65, 65, 1), (100, 300, 1)]
bad = 0
for h, w, s in SHAPES:
    rng = np.random.default_rng(h * 1000 + w)
    imgs = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
    imgs[1] = 255
    plan = fht.Plan(w, h, s, in_dtype="u8", acc_dtype="i32", batch=3)
    d = plan.describe()
    out = plan(torch.from_numpy(imgs).cuda())
    torch.cuda.synchronize()
    errs = []
    for bi in range(3):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], s, dtype=np.int32)
        for k in fht.QUADRANTS:
            got = out[k][bi].cpu().numpy()
            if not np.array_equal(got, ref[k]):
                nd = np.argwhere(got != ref[k])
                errs.append(f"{k}/img{bi}: {len(nd)} cells, first {nd[0].tolist()}")
    bad += bool(errs)
    info = [(g["quadrants"], g["u16_pair_D"], g["k2_tma_windows"], g["pass_rows"]) for g in d["groups"]]
    print(f"{h}x{w} s{s}: {'OK' if not errs else 'FAIL ' + '; '.join(errs[:4])}  {info}", flush=True)
print("bad shapes:", bad)
