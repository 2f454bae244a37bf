"""Small end-to-end run of every kernel family, for compute-sanitizer."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_07351_b200 import fht, shard  # noqa: E402

rng = np.random.default_rng(0)
for (h, w, strat, ind, acc) in [(77, 93, "tweaked", "u8", "i32"), (509, 509, "tweaked", "u8", "i32"),
                                (130, 257, "simple", "u8", "i32"), (64, 64, "tweaked", "f32", "f32"),
                                (45, 31, "tweaked", "i32", "i64"), (1, 40, "tweaked", "u8", "i32"),
                                (300, 1, "simple", "u8", "i32")]:
    if ind == "f32":
        img = rng.standard_normal((2, h, w)).astype(np.float32)
    else:
        img = rng.integers(0, 200, (2, h, w)).astype({"u8": np.uint8, "i32": np.int32}[ind])
    plan = fht.Plan(w, h, strat, in_dtype=ind, acc_dtype=acc, batch=2)
    out = plan(torch.from_numpy(img).cuda())
    plan.execute_host(img)
    nat = fht.Plan(w, h, strat, in_dtype=ind, acc_dtype=acc, batch=2, layout="native")(torch.from_numpy(img).cuda())
print(fht.fht2d_quadrants(rng.integers(-99, 99, (33, 41))).horiz_pos.shape)
x = torch.from_numpy(rng.integers(0, 255, (100, 129), dtype=np.uint8)).cuda()
print(fht.slow_hough_device(x, "vert_neg").shape)
be = shard.GpuRootBackend("tweaked", "u8", "i32")
print(shard.root_split_quadrant(x, "horiz_neg", "tweaked", side=0, backend=be, peer=None)[0].shape)
torch.cuda.synchronize()
print("ok")
