"""Randomised GPU sweep: seeded random shapes, strategies, dtypes, layouts,
quadrant masks and batch sizes, every result bit-exact against the oracle.
Exercises the plan paths the fixed cases miss (odd block remainders, bands of
different heights, carries, thin images, H below the row tile)."""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

Q = oracle.QUADRANTS


@pytest.mark.parametrize("seed", range(40))
def test_random_plans(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(6):
        h = int(rng.choice([1, 2, 3, 5, 31, 32, 33, 63, 64, 65, 127, 200, 257, 400, 700]))
        w = int(rng.choice([1, 2, 3, 17, 31, 32, 33, 64, 65, 96, 129, 255, 511, 600, 1025]))
        strategy = int(rng.integers(2))
        kind = rng.choice(["u8/i32", "u8/i64", "i32/i32", "i32/i64", "f32/f32", "u8/i32->i64"])
        layout = rng.choice(["reference", "native"])
        mask = int(rng.integers(1, 16))
        quads = [q for i, q in enumerate(Q) if mask & (1 << i)]
        b = int(rng.integers(1, 4))
        ind, rest = kind.split("/")
        acc, outd = (rest.split("->") + [None])[:2]
        if ind == "f32":
            imgs = rng.standard_normal((b, h, w)).astype(np.float32)
        elif ind == "i32":
            imgs = rng.integers(-30000, 30000, (b, h, w)).astype(np.int32)
        else:
            imgs = rng.integers(0, 256, (b, h, w)).astype(np.uint8)
        plan = fht.Plan(w, h, strategy, in_dtype=ind, acc_dtype=acc, out_dtype=outd, quadrants=quads, batch=b,
                        layout=layout)
        out = plan(torch.from_numpy(imgs).cuda())
        torch.cuda.synchronize()
        odt = {"i32": np.int32, "i64": np.int64, "f32": np.float32}[acc]
        for bi in range(b):
            ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=odt)
            for q in quads:
                got = out[q][bi].cpu().numpy()
                exp = ref[q] if layout == "reference" else ref[q].T
                assert np.array_equal(got, exp.astype(got.dtype)), (h, w, strategy, kind, layout, q, bi)


@pytest.mark.parametrize("strategy", [0, 1])
def test_every_narrow_width(strategy):
    """Every width 1..70 (all remainder-block shapes below and around one
    32-block, the K1 / K1P split, the first bands) at a few heights, all four
    quadrants, u8 -> i32, bit-exact against the oracle."""
    rng = np.random.default_rng(77 + strategy)
    for w in range(1, 71):
        for h in (1, 6, 37):
            imgs = rng.integers(0, 256, (2, h, w)).astype(np.uint8)
            plan = fht.Plan(w, h, strategy, in_dtype="u8", acc_dtype="i32", batch=2)
            out = plan(torch.from_numpy(imgs).cuda())
            torch.cuda.synchronize()
            for b in range(2):
                ref, _ = oracle.fht2d_quadrants(imgs[b], strategy, dtype=np.int32)
                for k in Q:
                    np.testing.assert_array_equal(out[k][b].cpu().numpy(), ref[k], err_msg=f"{h}x{w} {k} s{strategy}")
