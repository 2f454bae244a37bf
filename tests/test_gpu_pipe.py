"""GPU parity of the fused upper passes across their kernel variants: several
band layouts (non-root bands storing from registers, copy tiles, root bands
storing through shared memory) with the pair-mode root band's slots-per-CTA
setting and its double buffering switched on and off (FHT_K2_PIPE), against
the oracle."""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

Q = oracle.QUADRANTS


def _run(imgs, in_dtype, acc, strategy, quadrants="all"):
    b, h, w = imgs.shape
    plan = fht.Plan(w, h, strategy, in_dtype=in_dtype, acc_dtype=acc, quadrants=quadrants, batch=b)
    out = plan(torch.from_numpy(np.ascontiguousarray(imgs)).cuda())
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}, plan.describe()


CASES = [
    ((2, 700, 1500), "f32", "f32", 0),   # Simple: two bands (non-root + root), copy tiles
    ((1, 2100, 300), "i32", "i32", 1),   # two bands in the vertical orientation
    ((3, 1000, 1000), "u8", "i32", 1),   # one 5-level root band, 32-slope tiles
    ((2, 333, 271), "f32", "f32", 1),
]


@pytest.mark.parametrize("shape,ind,acc,strategy", CASES)
@pytest.mark.parametrize("ipc", ["1", "3"])
def test_pipe_bit_exact(monkeypatch, shape, ind, acc, strategy, ipc):
    monkeypatch.setenv("FHT_K2_SLOTS_PER_CTA", ipc)
    rng = np.random.default_rng(sum(shape))
    if ind == "f32":
        imgs = rng.standard_normal(shape).astype(np.float32)
        dt = np.float32
    elif ind == "i32":
        imgs = rng.integers(-5000, 5000, shape).astype(np.int32)
        dt = np.int32
    else:
        imgs = rng.integers(0, 256, shape, dtype=np.uint8)
        dt = np.int32
    out, desc = _run(imgs, ind, acc, strategy)
    for bi in range(shape[0]):
        ref, _ = oracle.fht2d_quadrants(imgs[bi], strategy, dtype=dt)
        for k in Q:
            np.testing.assert_array_equal(out[k][bi], ref[k], err_msg=f"{shape} {ind} s{strategy} {k} img{bi}")
    # the same bytes through the single-item kernel
    monkeypatch.setenv("FHT_K2_PIPE", "0")
    out0, _ = _run(imgs, ind, acc, strategy)
    for k in Q:
        np.testing.assert_array_equal(out0[k], out[k])
