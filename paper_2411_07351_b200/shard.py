"""Multi-GPU sharding of the FHT2D path: one process per GPU, no collective on
the data path.

* Batches (config c4): images are independent -> each rank transforms a
  contiguous, balanced shard of the batch (`batch_shard`).
* One large image (config c5): the four quadrants are independent -> rank r
  transforms the quadrants assigned to it (`quadrant_shard`).
* One large image on more ranks than quadrants (c5 on 8 GPUs): two GPUs per
  quadrant split its root (`image_assignment`, `root_split_quadrant`); the one exchange is fused into the child
  transform, whose last pass stores the slopes the peer needs straight into
  the peer's buffer over NVLink (`PeerExchange`, CUDA IPC), NCCL/gloo
  send/recv as the fallback.
* Results may optionally be gathered to rank 0 with one collective
  (`gather_to_root`, NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import os
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
    none (`image_assignment` pairs them up for a root split instead)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    return [q for i, q in enumerate(quadrants) if i % world == rank]


@dataclass(frozen=True)
class Assignment:
    """What one rank computes of a single large image: `quadrants` whole, or
    (when `side` is not None) one child subtree of `quadrants[0]`'s root,
    paired with rank `peer` (root_split_quadrant)."""
    quadrants: tuple
    side: int | None = None
    peer: int | None = None


def image_assignment(world: int, rank: int, quadrants=QUADRANTS) -> Assignment:
    """Work of `rank` for one image on `world` ranks, every quadrant owned:
    world <= Q: quadrants round-robin (quadrant_shard).  Q < world: the first
    world - Q quadrants (at most Q) get two ranks each and are root-split, the
    rest one rank each; ranks past 2Q idle.  E.g. Q = 4, world = 6: quadrants
    0 and 1 on ranks (0, 1) and (2, 3), quadrants 2 and 3 on ranks 4 and 5."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    nq = len(quadrants)
    if world <= nq:
        return Assignment(tuple(quadrant_shard(world, rank, quadrants)))
    split = min(nq, world - nq)  # quadrants that get a pair of ranks
    if rank < 2 * split:
        return Assignment((quadrants[rank // 2],), rank % 2, rank ^ 1)
    k = split + (rank - 2 * split)  # a single-rank quadrant, or idle
    return Assignment((quadrants[k],) if k < nq else ())


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


# ----------------------------------------------------------- root split
@dataclass(frozen=True)
class RootSplit:
    """Two GPUs share one quadrant of a large image (SURVEY §8e, config c5 on
    8 GPUs): side 0 computes the root's left child subtree (working columns
    [0, w0)), side 1 the right child ([w0, W)); they swap the child columns
    the other side needs and each merges half of the root's slopes:
    side 0 slopes [0, t_mid), side 1 [t_mid, W) (transform.cpp:46-57)."""
    W: int
    H: int
    w0: int
    w1: int
    t_mid: int
    right_for_0: tuple  # right-child slopes [lo, hi) side 1 sends to side 0
    left_for_1: tuple   # left-child slopes [lo, hi) side 0 sends to side 1


def root_split(W: int, H: int, strategy) -> RootSplit:
    from .fht import round_half_up_ratio, split_width

    if W < 2:
        raise ValueError("root split needs width >= 2")
    w0, w1 = split_width(W, strategy)
    t_mid = W // 2

    def t0(t):
        return round_half_up_ratio(t * (w0 - 1), W - 1)

    def t1(t):
        return round_half_up_ratio(t * (w1 - 1), W - 1)

    return RootSplit(W, H, w0, w1, t_mid, (t1(0), t1(t_mid - 1) + 1), (t0(t_mid), t0(W - 1) + 1))


def child_view(img, quadrant: str, side: int, split: RootSplit):
    """The sub-image whose `quadrant` transform is the root's child `side`
    (a view: rows keep the parent's pitch).  Returns the 2-D view."""
    h, w = img.shape
    x0, cw = (0, split.w0) if side == 0 else (split.w0, split.w1)
    if quadrant == "horiz_pos":
        return img[:, x0:x0 + cw]
    if quadrant == "horiz_neg":
        return img[:, w - x0 - cw:w - x0]
    if quadrant == "vert_pos":
        return img[x0:x0 + cw, :]
    if quadrant == "vert_neg":
        return img[h - x0 - cw:h - x0, :]
    raise ValueError(quadrant)


class GpuRootBackend:
    """Child transforms with a pitched plan (fht_execute_pitched, slope-major
    output) and the root merge kernel (fht_merge_root)."""

    def __init__(self, strategy, in_dtype: str, acc_dtype: str, out_dtype: str | None = None, layout="reference"):
        self.strategy, self.in_dtype, self.acc_dtype = strategy, in_dtype, acc_dtype
        self.out_dtype = out_dtype or acc_dtype
        self.layout = layout
        self._plans = {}

    def child(self, view, quadrant: str, side: int = 0, peer_ptr: int | None = None, peer_cols=(0, 0)):
        import ctypes

        import torch

        from . import fht
        from ._lib import check, lib

        h, w = view.shape
        key = (w, h, quadrant, side, view.device.index or 0)  # per side: loopback keeps both children
        if key not in self._plans:  # plans (tables, workspace, outputs) are built once per shape
            plan = fht.Plan(w, h, self.strategy, in_dtype=self.in_dtype, acc_dtype=self.acc_dtype,
                            quadrants=[quadrant], layout="native", device=view.device.index or 0)
            self._plans[key] = (plan, plan.alloc_outputs(), plan.workspace())
        plan, out, ws = self._plans[key]
        ptrs = (ctypes.c_void_p * 4)()
        ptrs[fht.QUADRANTS.index(quadrant)] = out[quadrant].data_ptr()
        st = torch.cuda.current_stream(view.device)
        wsp = ctypes.c_void_p(ws.data_ptr() if ws is not None else 0)
        if peer_ptr:  # the exchange fused into the last pass: peer slopes stored over NVLink
            check(lib().fht_execute_pitched_peer(plan._h, ctypes.c_void_p(view.data_ptr()), view.stride(0), ptrs, wsp,
                                                 ctypes.c_void_p(peer_ptr), int(peer_cols[0]), int(peer_cols[1]),
                                                 ctypes.c_void_p(st.cuda_stream)))
        else:
            check(lib().fht_execute_pitched(plan._h, ctypes.c_void_p(view.data_ptr()), view.stride(0), 0, ptrs, 0, wsp,
                                            ctypes.c_void_p(st.cuda_stream)))
        return out[quadrant][0]  # (child width, H) slope-major

    def peer_exchange(self, key, nbytes: int, device: int, peer: int, group=None) -> "PeerExchange":
        """The receive buffer this side exposes to its root-split peer and the
        peer's buffer mapped here (CUDA IPC over NVLink), built once per key."""
        if not hasattr(self, "_peers"):
            self._peers = {}
        if key not in self._peers:
            import torch.distributed as dist

            # the store tag both ranks of the pair derive alike: the pair and
            # the quadrant / shape (not the side, which differs between them)
            quadrant, _side, W, H = key
            pair = "-".join(str(r) for r in sorted((dist.get_rank(), peer)))
            self._peers[key] = PeerExchange(nbytes, device, peer, group, key=f"{pair}/{quadrant}/{W}x{H}")
        return self._peers[key]

    def merge(self, split: RootSplit, left, left_first, right, right_first, t_beg, t_end, out):
        import ctypes

        import torch

        from . import fht
        from ._lib import check, lib

        st = torch.cuda.current_stream(out.device)
        lp = left if isinstance(left, int) else left.data_ptr()  # tensors, or raw device pointers
        rp = right if isinstance(right, int) else right.data_ptr()
        check(lib().fht_merge_root(split.W, split.H, fht._strategy(self.strategy), fht._dtype_code(self.acc_dtype),
                                   fht._dtype_code(self.out_dtype), 0 if self.layout == "reference" else 1,
                                   ctypes.c_void_p(lp), left_first, ctypes.c_void_p(rp), right_first, t_beg, t_end,
                                   ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))

    def empty_out(self, split: RootSplit, like, key=None):
        """The root output buffer: full size, each side writes only its own
        slopes.  With a `key` it is allocated once and reused every step (the
        other side's slopes are left as they are -- uninitialised)."""
        import torch

        dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32}[self.out_dtype]
        shape = (split.H, split.W) if self.layout == "reference" else (split.W, split.H)
        if key is None:
            return torch.zeros(shape, dtype=dt, device=like.device)
        if not hasattr(self, "_outs"):
            self._outs = {}
        if key not in self._outs:
            self._outs[key] = torch.empty(shape, dtype=dt, device=like.device)
        return self._outs[key]


class PeerExchange:
    """One side's half of the fused root-split exchange: a dedicated device
    buffer the peer writes its child slopes into (exported as a CUDA IPC
    handle), and the peer's buffer opened here.  Handles travel once over the
    process group (any backend); the data never does -- the child transform's
    last pass stores it straight into peer memory over NVLink.

    Per step the two sides are ordered on the device, with no stream
    synchronisation and no collective: two interprocess CUDA events per side
    ("my peer stores have landed", "I am done reading my receive buffer"),
    waited with cudaStreamWaitEvent on the other side.  cudaStreamWaitEvent
    binds to an event's most recent record, so a side must not wait before
    the peer has *issued* this step's record: two host counters in a shared
    memory segment (the ranks of a pair share a node) carry "record k issued"
    -- a host flag, not a device sync; the GPU queue keeps running ahead."""

    TIMEOUT_S = 120.0

    def __init__(self, nbytes: int, device: int, peer: int, group=None, key: str = "0"):
        import ctypes

        import torch
        import torch.distributed as dist

        from ._lib import check, lib

        self.key = key
        self.local = ctypes.c_void_p()
        check(lib().fht_device_alloc(max(1, nbytes), device, ctypes.byref(self.local)))
        handle = ctypes.create_string_buffer(64)
        check(lib().fht_ipc_get_handle(self.local, handle, 64))
        self.rank, self.peer = dist.get_rank(), peer
        self.side = 0 if self.rank < peer else 1
        self.dev = torch.device("cuda", device)
        # my events: 0 = peer stores issued by me have landed, 1 = my receive buffer is free
        self.ev = [torch.cuda.Event(enable_timing=False, blocking=False, interprocess=True) for _ in range(2)]
        for e in self.ev:
            e.record(torch.cuda.current_stream(self.dev))  # an IPC handle needs a recorded event
        torch.cuda.current_stream(self.dev).synchronize()
        shm_name = None
        if self.side == 0:
            from multiprocessing import shared_memory

            self._shm = shared_memory.SharedMemory(create=True, size=64)
            shm_name = self._shm.name
        # the handles travel through the process group's key-value store: only
        # the two ranks of the pair take part (other ranks may be doing other
        # work, e.g. a quadrant of their own)
        import pickle

        from torch.distributed import distributed_c10d as c10d

        store = c10d._get_default_store()  # noqa: SLF001
        tag = f"fht_root_split/{self.key}"
        store.set(f"{tag}/{self.rank}", pickle.dumps((handle.raw, [e.ipc_handle() for e in self.ev], shm_name)))
        peer_handle, peer_ev, peer_shm = pickle.loads(store.get(f"{tag}/{peer}"))
        self.remote = ctypes.c_void_p()
        check(lib().fht_ipc_open_handle(peer_handle, 64, device, ctypes.byref(self.remote)))
        self.peer_ev = [torch.cuda.Event.from_ipc_handle(self.dev, h) for h in peer_ev]
        if self.side == 1:
            from multiprocessing import resource_tracker, shared_memory

            self._shm = shared_memory.SharedMemory(name=peer_shm)
            # the creator (side 0) owns the segment's lifetime
            resource_tracker.unregister(self._shm._name, "shared_memory")  # noqa: SLF001
        import numpy as np

        # counters[side * 2 + e]: the step whose record of event e that side has issued
        self.counters = np.ndarray((4,), dtype=np.int64, buffer=self._shm.buf)
        if self.side == 0:
            self.counters[:] = 0
        self.step = 0

    def _await(self, who: int, e: int, k: int):
        import time

        t0 = time.monotonic()
        spins = 0
        while self.counters[who * 2 + e] < k:
            spins += 1
            if spins > 1000:
                time.sleep(0)
                if time.monotonic() - t0 > self.TIMEOUT_S:
                    raise RuntimeError("root split: the peer stopped responding")

    def begin(self, stream):
        """Before this step's child transform writes into the peer's buffer:
        wait (on the device) until the peer has finished reading it."""
        self.step += 1
        if self.step > 1:
            self._await(1 - self.side, 1, self.step - 1)
            stream.wait_event(self.peer_ev[1])

    def stored(self, stream):
        """After the child transform: publish "my stores into the peer landed"
        and wait (on the device) for the peer's stores into my buffer."""
        self.ev[0].record(stream)
        self.counters[self.side * 2] = self.step
        self._await(1 - self.side, 0, self.step)
        stream.wait_event(self.peer_ev[0])

    def consumed(self, stream):
        """After the merge: my receive buffer may be overwritten again."""
        self.ev[1].record(stream)
        self.counters[self.side * 2 + 1] = self.step

    def close(self):
        from ._lib import lib

        if self.remote:
            lib().fht_ipc_close(self.remote)
            self.remote = None
        if self.local:
            lib().fht_device_free(self.local)
            self.local = None
        shm = getattr(self, "_shm", None)
        if shm is not None:
            self.counters = None
            shm.close()
            if self.side == 0:
                shm.unlink()
            self._shm = None


def root_split_quadrant(img, quadrant: str, strategy, side: int, backend, peer: int | None = None, group=None,
                        exchange: str | None = None):
    """One side of the two-GPU root split of `quadrant` of `img` (the whole
    image, resident on this rank).  `peer` is the other side's global rank
    (None: both sides run in this process, `side` ignored -- used to test the
    kernels on one GPU).  Returns this side's output buffer (full size, the
    slopes this side merged filled in) and the split description."""
    import torch
    import torch.distributed as dist

    horiz = quadrant.startswith("horiz")
    h, w = img.shape
    W, H = (w, h) if horiz else (h, w)
    sp = root_split(W, H, strategy)
    if peer is None:  # loopback: both children and both halves here
        left = backend.child(child_view(img, quadrant, 0, sp), quadrant, 0)
        right = backend.child(child_view(img, quadrant, 1, sp), quadrant, 1)
        out = backend.empty_out(sp, left)
        backend.merge(sp, left, 0, right, 0, 0, W, out)
        return out, sp
    lo, hi = sp.left_for_1 if side == 0 else sp.right_for_0
    rlo, rhi = sp.right_for_0 if side == 0 else sp.left_for_1
    exchange = exchange or os.environ.get("FHT_ROOT_EXCHANGE", "p2p")
    if exchange == "p2p" and img.is_cuda and hasattr(backend, "peer_exchange"):
        # The exchange fused into the child transform: its last pass stores
        # the slopes the peer needs straight into the peer's buffer (CUDA IPC
        # mapping, NVLink stores); two barriers order the steps.
        dev = img.device.index or 0
        esz = torch.empty((), dtype={"i32": torch.int32, "i64": torch.int64, "f32": torch.float32}[backend.acc_dtype]
                          ).element_size()
        ex = backend.peer_exchange((quadrant, side, W, H), max(rhi - rlo, hi - lo) * H * esz, dev, peer, group)
        st = torch.cuda.current_stream(img.device)
        ex.begin(st)  # device wait: the peer is done reading its buffer from the previous step
        mine = backend.child(child_view(img, quadrant, side, sp), quadrant, side, peer_ptr=ex.remote.value,
                             peer_cols=(lo, hi))
        ex.stored(st)  # device wait: the peer's stores into my buffer have landed
        out = backend.empty_out(sp, mine, key=(quadrant, side, W, H))
        if side == 0:
            backend.merge(sp, mine, 0, ex.local.value, rlo, 0, sp.t_mid, out)
        else:
            backend.merge(sp, ex.local.value, rlo, mine, 0, sp.t_mid, W, out)
        ex.consumed(st)
        return out, sp
    mine = backend.child(child_view(img, quadrant, side, sp), quadrant, side)
    # gloo moves host tensors only: stage the exchange through host memory
    # (NCCL exchanges device buffers directly over NVLink)
    host = dist.get_backend(group) == "gloo" and mine.device.type == "cuda"
    send = mine[lo:hi].contiguous()
    recv = torch.empty((rhi - rlo, H), dtype=mine.dtype, device=mine.device)
    send_x, recv_x = (send.cpu(), torch.empty(recv.shape, dtype=recv.dtype)) if host else (send, recv)
    if side == 0:
        ops = [dist.P2POp(dist.isend, send_x, peer, group), dist.P2POp(dist.irecv, recv_x, peer, group)]
    else:
        ops = [dist.P2POp(dist.irecv, recv_x, peer, group), dist.P2POp(dist.isend, send_x, peer, group)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    if host:
        recv.copy_(recv_x)
    out = backend.empty_out(sp, mine)
    if side == 0:
        backend.merge(sp, mine, 0, recv, rlo, 0, sp.t_mid, out)
    else:
        backend.merge(sp, recv, rlo, mine, 0, sp.t_mid, W, out)
    return out, sp
