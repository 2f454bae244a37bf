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
