"""CPU (gloo, world_size 2) tests of the multi-GPU host logic: every image is
transformed by exactly one rank, and gathering the per-rank results
reproduces the single-process transform of the whole batch (the transform
here is the oracle, since this container has no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_07351_b200.shard import (QUADRANTS, batch_shard, gather_to_root, image_assignment, max_over_ranks,
                                         quadrant_shard)


def test_batch_shard_covers_exactly_once():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                s = batch_shard(n, world, r)
                seen.extend(range(s.start, s.start + s.count))
            assert seen == list(range(n))
            counts = [batch_shard(n, world, r).count for r in range(world)]
            assert max(counts) - min(counts) <= 1


def test_quadrant_shard():
    assert [quadrant_shard(4, r) for r in range(4)] == [[q] for q in QUADRANTS]
    assert sorted(sum((quadrant_shard(2, r) for r in range(2)), [])) == sorted(QUADRANTS)
    assert sum((quadrant_shard(8, r) for r in range(8)), []) == list(QUADRANTS)
    with pytest.raises(ValueError):
        batch_shard(4, 2, 2)


@pytest.mark.parametrize("world", range(1, 11))
def test_image_assignment_owns_every_quadrant(world):
    """Every quadrant of a single image is computed for any world size: whole
    by one rank, or root-split by a pair of ranks that name each other."""
    owners = {q: [] for q in QUADRANTS}
    for r in range(world):
        a = image_assignment(world, r)
        for q in a.quadrants:
            owners[q].append((r, a.side, a.peer))
    for q, own in owners.items():
        assert own, (world, q)
        if len(own) == 1:
            assert own[0][1] is None
        else:
            assert len(own) == 2
            (r0, s0, p0), (r1, s1, p1) = own
            assert {s0, s1} == {0, 1} and p0 == r1 and p1 == r0
    busy = sum(1 for r in range(world) if image_assignment(world, r).quadrants)
    assert busy == min(world, 2 * len(QUADRANTS))
    if world == 8:
        assert all(image_assignment(8, r).side == r % 2 for r in range(8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    rng = np.random.default_rng(5)
    imgs = rng.integers(0, 256, (6, 23, 31), dtype=np.uint8)  # same batch on every rank
    sh = batch_shard(len(imgs), world, rank)
    res = []
    for i in range(sh.start, sh.start + sh.count):
        q, _ = oracle.fht2d_quadrants(imgs[i], oracle.TWEAKED, dtype=np.int32)
        res.append(np.stack([q["horiz_pos"], q["horiz_neg"]]))
    local = torch.from_numpy(np.stack(res))
    full = gather_to_root(local)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(out_path, full.numpy())
        assert t == float(world)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_matches_single_process(tmp_path):
    world, out = 2, tmp_path / "gathered.npy"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    import oracle

    rng = np.random.default_rng(5)
    imgs = rng.integers(0, 256, (6, 23, 31), dtype=np.uint8)
    ref = []
    for i in range(6):
        q, _ = oracle.fht2d_quadrants(imgs[i], oracle.TWEAKED, dtype=np.int32)
        ref.append(np.stack([q["horiz_pos"], q["horiz_neg"]]))
    np.testing.assert_array_equal(np.load(out), np.stack(ref))


# ------------------------------------------------------------ root split
class _CpuRootBackend:
    """The root split driven by the oracle on CPU tensors (no GPU here)."""

    def __init__(self, strategy):
        self.strategy = strategy

    def child(self, view, quadrant, side=0):
        import oracle

        v = view.numpy()
        q, _ = oracle.fht2d_quadrants(np.ascontiguousarray(v), self.strategy, dtype=np.int64)
        return torch.from_numpy(np.ascontiguousarray(q[quadrant].T))  # slope-major (W_child, H)

    def merge(self, sp, left, left_first, right, right_first, t_beg, t_end, out):
        from paper_2411_07351_b200.fht import round_half_up_ratio

        for t in range(t_beg, t_end):
            t0 = round_half_up_ratio(t * (sp.w0 - 1), sp.W - 1)
            t1 = round_half_up_ratio(t * (sp.w1 - 1), sp.W - 1)
            r = (t - t1) % sp.H
            out[:, t] = left[t0 - left_first] + torch.roll(right[t1 - right_first], -r)

    def empty_out(self, sp, like):
        return torch.zeros((sp.H, sp.W), dtype=torch.int64)


def _root_worker(rank, world, port, out_path, quadrant, strategy):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_07351_b200.shard import root_split_quadrant

    rng = np.random.default_rng(11)
    img = torch.from_numpy(rng.integers(0, 1000, (37, 45)).astype(np.int64))
    out, sp = root_split_quadrant(img, quadrant, strategy, side=rank, backend=_CpuRootBackend(strategy), peer=1 - rank)
    np.save(f"{out_path}.{rank}.npy", out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("quadrant,strategy", [("horiz_pos", 1), ("horiz_neg", 0), ("vert_pos", 1), ("vert_neg", 1)])
def test_root_split_two_ranks_gloo(tmp_path, quadrant, strategy):
    import oracle
    from paper_2411_07351_b200.shard import root_split

    out = tmp_path / "root"
    mp.spawn(_root_worker, args=(2, _free_port(), str(out), quadrant, strategy), nprocs=2, join=True)
    rng = np.random.default_rng(11)
    img = rng.integers(0, 1000, (37, 45)).astype(np.int64)
    ref, _ = oracle.fht2d_quadrants(img, strategy)
    a, b = np.load(f"{out}.0.npy"), np.load(f"{out}.1.npy")
    H, W = ref[quadrant].shape
    sp = root_split(W, H, strategy)
    np.testing.assert_array_equal(a[:, :sp.t_mid], ref[quadrant][:, :sp.t_mid])
    np.testing.assert_array_equal(b[:, sp.t_mid:], ref[quadrant][:, sp.t_mid:])
