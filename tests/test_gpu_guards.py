"""Out-of-bounds write guards (compute-sanitizer is closed on the GPU pool).

Every output quadrant and the workspace are views into larger buffers whose
margins hold a sentinel; after the transform the margins must be untouched
and the results bit-exact against the oracle (transform.cpp:62-85,
quadrants.cpp:23-41).  The shapes cover the kernel families: the u16 pair
mode with TMA windows (509^2, the c4 shape), K1P + generic K1 tail blocks,
Simple splits, one-row / one-column images, float32, int32 -> int64
widening, the native layout and several images per plan.
"""
import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

PAD = 4096  # bytes of margin on each side
SENT = 0x5A

CASES = [
    # (h, w, strategy, in, acc, out, layout, batch)
    (509, 509, "tweaked", "u8", "i32", None, "reference", 3),  # pair mode, TMA windows
    (509, 509, "tweaked", "u8", "i32", None, "native", 2),
    (77, 93, "tweaked", "u8", "i32", None, "reference", 2),
    (130, 257, "simple", "u8", "i32", None, "reference", 1),
    (1, 40, "tweaked", "u8", "i32", None, "reference", 2),
    (300, 1, "simple", "u8", "i32", None, "reference", 1),
    (64, 64, "tweaked", "f32", "f32", None, "reference", 2),
    (45, 31, "tweaked", "i32", "i32", "i64", "reference", 2),
    (333, 200, "tweaked", "i32", "i64", None, "reference", 1),
    (600, 700, "simple", "u8", "i32", None, "reference", 1),
]


def _guarded(nbytes, dev):
    big = torch.full((nbytes + 2 * PAD,), SENT, dtype=torch.uint8, device=dev)
    return big, big[PAD:PAD + nbytes]


def _margins_intact(big):
    b = big.cpu().numpy()
    return bool((b[:PAD] == SENT).all() and (b[-PAD:] == SENT).all())


@pytest.mark.parametrize("h,w,strategy,ind,acc,outd,layout,batch", CASES)
def test_no_writes_outside_outputs_and_workspace(h, w, strategy, ind, acc, outd, layout, batch):
    rng = np.random.default_rng(h * 1000 + w)
    np_dt = {"u8": np.uint8, "i32": np.int32, "f32": np.float32}[ind]
    if ind == "f32":
        imgs = rng.standard_normal((batch, h, w)).astype(np.float32)
    else:
        imgs = rng.integers(0, 200, (batch, h, w)).astype(np_dt)
    plan = fht.Plan(w, h, strategy, in_dtype=ind, acc_dtype=acc, out_dtype=outd, batch=batch, layout=layout)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    # the workspace the plan will use on this stream: a guarded view
    ws_big = None
    if plan.workspace_bytes:
        ws_big, ws = _guarded(plan.workspace_bytes, dev)
        plan._ws[int(st.cuda_stream)] = ws
    tdt = plan._torch_dtype(plan.out_dtype)
    esz = torch.empty((), dtype=tdt).element_size()
    bigs, out = {}, {}
    for q in plan.quadrants:
        shape = (batch, *plan.out_shape(q))
        n = int(np.prod(shape)) * esz
        big, view = _guarded(n, dev)
        bigs[q] = big
        out[q] = view.view(tdt).view(shape)
    plan(torch.from_numpy(imgs).cuda(), out)
    torch.cuda.synchronize()
    for q, big in bigs.items():
        assert _margins_intact(big), f"write outside output {q}"
    if ws_big is not None:
        assert _margins_intact(ws_big), "write outside the workspace"
    strat = oracle.TWEAKED if strategy == "tweaked" else oracle.SIMPLE
    ref_dt = {"u8": np.int32, "i32": np.int64 if acc == "i64" else np.int32, "f32": np.float32}[ind]
    if ind == "i32" and outd == "i64":
        ref_dt = np.int64
    for b in range(batch):
        ref, _ = oracle.fht2d_quadrants(imgs[b], strat, dtype=ref_dt)
        for q in plan.quadrants:
            got = out[q][b].cpu().numpy()
            want = ref[q] if layout == "reference" else ref[q].T
            np.testing.assert_array_equal(got, want.astype(got.dtype))
