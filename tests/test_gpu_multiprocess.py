"""The multi-rank GPU paths with real kernels: several processes share the one
GPU of the test box over a gloo process group (their kernels never wait on
each other; only host-side collectives).  Checks the two-rank root split of a
quadrant against the single-process transform, and runs bench.py under
torchrun with 2 ranks (batch shards) and 8 ranks (c5-style root split)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _root_worker(rank, port, out, exchange):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FHT_ROOT_EXCHANGE=exchange)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    sys.path.insert(0, str(ROOT))
    from paper_2411_07351_b200 import shard

    from paper_2411_07351_b200 import _lib

    be = shard.GpuRootBackend("tweaked", "f32", "f32")
    imgs = [torch.from_numpy(np.random.default_rng(9 + k).random((1500, 2049), dtype=np.float32)).cuda()
            for k in range(3)]
    for k in range(3):  # three steps, a new image each: buffers, events and counters are reused across steps
        if k == 1:  # after the first step (plans, buffers, IPC set up): no allocation, no host sync
            c0 = _lib.debug_counters()
            a0 = torch.cuda.memory_stats()["allocation.all.allocated"]
        res, sp = shard.root_split_quadrant(imgs[k], "vert_pos", "tweaked", side=rank, backend=be, peer=1 - rank)
    if exchange == "p2p":
        assert _lib.debug_counters() == c0, (c0, _lib.debug_counters())
        assert torch.cuda.memory_stats()["allocation.all.allocated"] == a0
    torch.cuda.synchronize()
    np.save(f"{out}.{rank}.npy", res.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["p2p", "sendrecv"])
def test_root_split_two_processes_one_gpu(tmp_path, exchange):
    """p2p: the children store the peer's slopes through a CUDA IPC mapping of
    the peer process's buffer (the fused exchange); sendrecv: the fallback."""
    import torch.multiprocessing as mp

    from paper_2411_07351_b200 import fht, shard

    out = tmp_path / "rs"
    mp.spawn(_root_worker, args=(_port(), str(out), exchange), nprocs=2, join=True)
    rng = np.random.default_rng(11)  # the last step's image
    img = torch.from_numpy(rng.random((1500, 2049), dtype=np.float32)).cuda()
    full = fht.Plan(2049, 1500, "tweaked", in_dtype="f32", acc_dtype="f32", quadrants=["vert_pos"])(img[None])
    ref = full["vert_pos"][0].cpu().numpy()
    sp = shard.root_split(1500, 2049, "tweaked")
    a, b = np.load(f"{out}.0.npy"), np.load(f"{out}.1.npy")
    np.testing.assert_array_equal(a[:, :sp.t_mid], ref[:, :sp.t_mid])
    np.testing.assert_array_equal(b[:, sp.t_mid:], ref[:, sp.t_mid:])


def _torchrun(n, *args):
    env = dict(os.environ, FHT_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", str(n),
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_two_ranks_batch_shards():
    """BASELINE c4 on N GPUs: the one 256-image batch sharded 128 + 128."""
    d = _torchrun(2)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("batch-shard x2") and d["config"]["images_per_gpu"] == 128
    assert d["images_per_s"] == pytest.approx(256 / (d["ms_per_step"] * 1e-3), rel=1e-2)
    w = d["weak_scaling"]
    assert w["images_per_gpu"] == 256 and w["value"] > 0


def test_bench_two_ranks_weak():
    d = _torchrun(2, "--scaling", "weak", "--no-weak")
    assert d["scaling"] == "weak" and d["config"]["images_per_gpu"] == 256 and d["weak_scaling"] is None


def test_bench_six_ranks_every_quadrant_owned():
    """6 ranks on one image: two quadrants root-split, two whole (image_assignment)."""
    d = _torchrun(6, "--config", "c3", "--no-weak")
    assert d["n_gpus"] == 6 and d["scaling"] == "strong" and d["value"] > 0


def test_bench_eight_ranks_root_split_c5():
    d = _torchrun(8, "--config", "c5")
    assert d["n_gpus"] == 8 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["parallelism"] == "root-split x2 per quadrant"
