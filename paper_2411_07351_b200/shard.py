"""Multi-GPU sharding of the FHT2D path: one process per GPU, no collective on
the data path.

* Batches (config c4): images are independent -> each rank transforms a
  contiguous, balanced shard of the batch (`batch_shard`).
* One large image (config c5): the four quadrants are independent -> rank r
  transforms the quadrants assigned to it (`quadrant_shard`).
* Results may optionally be gathered to rank 0 with one collective
  (`gather_to_root`, NCCL on GPUs, gloo in the CPU tests).  The transform
  itself never communicates.
"""
from __future__ import annotations

from dataclasses import dataclass

QUADRANTS = ("horiz_pos", "horiz_neg", "vert_pos", "vert_neg")


@dataclass(frozen=True)
class Shard:
    start: int
    count: int


def batch_shard(n_items: int, world: int, rank: int) -> Shard:
    """Balanced contiguous split of n_items over `world` ranks (the first
    n_items % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    if n_items < 0:
        raise ValueError("n_items must be >= 0")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return Shard(start, base + (1 if rank < extra else 0))


def quadrant_shard(world: int, rank: int, quadrants=QUADRANTS) -> list[str]:
    """Quadrants of one image owned by `rank`: round-robin, so 4 ranks get one
    each, 2 ranks two each; with more ranks than quadrants the extra ranks get
    none (a root split of one quadrant over two GPUs is future work)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    return [q for i, q in enumerate(quadrants) if i % world == rank]


def gather_to_root(tensor, group=None, dst: int = 0):
    """Gather equally-shaped per-rank result tensors to `dst` (None elsewhere).
    Uses all_gather (supported by both NCCL and gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [torch.empty_like(tensor) for _ in range(world)]
    dist.all_gather(parts, tensor.contiguous(), group=group)
    return torch.cat(parts, dim=0) if dist.get_rank(group) == dst else None


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
