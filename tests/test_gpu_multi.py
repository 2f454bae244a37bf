"""GPU kernels of the multi-GPU paths on one device: pitched child plans +
the root-merge kernel (the two-GPU root split run as a loopback), and batch
shards equal to the unsharded batch."""
import numpy as np
import pytest

from paper_2411_07351_b200 import fht, shard, workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def _full(img, quadrant, strategy, in_dtype, acc):
    h, w = img.shape
    plan = fht.Plan(w, h, strategy, in_dtype=in_dtype, acc_dtype=acc, quadrants=[quadrant])
    return plan(img[None])[quadrant][0]


@pytest.mark.parametrize("quadrant", fht.QUADRANTS)
@pytest.mark.parametrize("strategy", ["tweaked", "simple"])
def test_root_split_loopback_int(quadrant, strategy):
    rng = np.random.default_rng(3)
    img = torch.from_numpy(rng.integers(0, 256, (1500, 2049), dtype=np.uint8)).cuda()
    be = shard.GpuRootBackend(strategy, "u8", "i32")
    out, sp = shard.root_split_quadrant(img, quadrant, strategy, side=0, backend=be, peer=None)
    torch.cuda.synchronize()
    assert torch.equal(out, _full(img, quadrant, strategy, "u8", "i32"))


@pytest.mark.parametrize("quadrant,strategy,in_dtype,acc", [("horiz_pos", "tweaked", "u8", "i32"),
                                                             ("vert_neg", "simple", "u8", "i32"),
                                                             ("vert_pos", "tweaked", "f32", "f32")])
def test_root_split_peer_stores(quadrant, strategy, in_dtype, acc):
    """The fused exchange: each child's last pass stores the slopes the other
    side needs straight into that side's receive buffer (here both sides in
    one process on one GPU, so a plain device pointer stands in for the IPC
    mapping); each side then merges its half of the root from its own child
    and the received slopes.  Equal to the single-plan transform."""
    rng = np.random.default_rng(4)
    if in_dtype == "u8":
        img = torch.from_numpy(rng.integers(0, 256, (1201, 1500), dtype=np.uint8)).cuda()
    else:
        img = torch.from_numpy(rng.random((1201, 1500), dtype=np.float32)).cuda()
    be = shard.GpuRootBackend(strategy, in_dtype, acc)
    h, w = img.shape
    W, H = (w, h) if quadrant.startswith("horiz") else (h, w)
    sp = shard.root_split(W, H, strategy)
    dt = {"i32": torch.int32, "f32": torch.float32}[acc]
    recv = [torch.full((sp.right_for_0[1] - sp.right_for_0[0], H), -7, dtype=dt, device="cuda"),  # side 0's
            torch.full((sp.left_for_1[1] - sp.left_for_1[0], H), -7, dtype=dt, device="cuda")]   # side 1's
    kids = []
    for side in (0, 1):
        cols = sp.left_for_1 if side == 0 else sp.right_for_0
        kids.append(be.child(shard.child_view(img, quadrant, side, sp), quadrant, side,
                             peer_ptr=recv[1 - side].data_ptr(), peer_cols=cols).clone())
    torch.cuda.synchronize()
    assert torch.equal(recv[0], kids[1][sp.right_for_0[0]:sp.right_for_0[1]])
    assert torch.equal(recv[1], kids[0][sp.left_for_1[0]:sp.left_for_1[1]])
    out = be.empty_out(sp, kids[0])
    be.merge(sp, kids[0], 0, recv[0].data_ptr(), sp.right_for_0[0], 0, sp.t_mid, out)
    be.merge(sp, recv[1].data_ptr(), sp.left_for_1[0], kids[1], 0, sp.t_mid, W, out)
    torch.cuda.synchronize()
    assert torch.equal(out, _full(img, quadrant, strategy, in_dtype, acc))


def test_root_split_loopback_float_c5_size():
    img = torch.from_numpy(workloads.make_images("c5", 1)[0]).cuda()
    be = shard.GpuRootBackend("tweaked", "f32", "f32")
    for q in ("horiz_pos", "vert_neg"):
        out, sp = shard.root_split_quadrant(img, q, "tweaked", side=0, backend=be, peer=None)
        torch.cuda.synchronize()
        assert sp.w0 == 4096 and sp.w1 == 4095
        assert torch.equal(out, _full(img, q, "tweaked", "f32", "f32"))  # same add tree: bit-exact


def test_batch_shards_equal_whole_batch():
    imgs = torch.from_numpy(workloads.make_images("c4", 12)).cuda()
    whole = fht.Plan(509, 509, "tweaked", in_dtype="u8", acc_dtype="i32", batch=12)(imgs)
    for world in (2, 3, 4):
        for r in range(world):
            sh = shard.batch_shard(12, world, r)
            if sh.count == 0:
                continue
            part = fht.Plan(509, 509, "tweaked", in_dtype="u8", acc_dtype="i32", batch=sh.count)(
                imgs[sh.start:sh.start + sh.count].contiguous())
            for q in fht.QUADRANTS:
                assert torch.equal(part[q], whole[q][sh.start:sh.start + sh.count])
