"""Python host API over the C ABI, mirroring the reference's C++ interface.

Reference (namespace fht, /root/reference/proj/include/fht):
  SplitStrategy            split.hpp:12-15     -> SplitStrategy
  split_simple/_tweaked/_width, round_half_up_ratio  split.hpp:33-57
  fht2d(img, strategy)     transform.hpp:36    -> fht2d
  fht2d_counted            transform.hpp:40    -> fht2d_counted (CountedTransform)
  fht2d_quadrants          quadrants.hpp:32-33 -> fht2d_quadrants (QuadrantSet)
  check_overflow_budget    transform.hpp:17    -> check_overflow_budget
  count_additions_tree     oracle.hpp:22       -> count_additions_tree

Images are numpy arrays of shape (h, w), row-major with x fastest, i.e. the
reference's data[y*w + x] (image.hpp:13-14).  Hough images come back in the
reference layout, shape (h, w) with J[s, t] = hough(t, s) (transform.cpp:80-83).

``Plan`` is the device-resident, batched API (the C ABI's fht_plan_*): it
takes torch CUDA tensors and never touches host memory.
"""
from __future__ import annotations

import ctypes
import enum
import json
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import FHT_F32, FHT_I32, FHT_I64, FHT_U8, InvalidArgument, OverflowBudget, check, lib

QUADRANTS = ("horiz_pos", "horiz_neg", "vert_pos", "vert_neg")


class SplitStrategy(enum.IntEnum):
    Simple = 0
    Tweaked = 1


def strategy_from_string(name: str) -> SplitStrategy:
    """split.hpp:21-25"""
    if name == "simple":
        return SplitStrategy.Simple
    if name == "tweaked":
        return SplitStrategy.Tweaked
    raise InvalidArgument(f"unknown strategy '{name}' (expected simple|tweaked)")


def _strategy(s) -> int:
    if isinstance(s, str):
        return int(strategy_from_string(s))
    s = int(s)
    if s not in (0, 1):
        raise InvalidArgument("unknown strategy")
    return s


_DT = {"u8": FHT_U8, "uint8": FHT_U8, "i32": FHT_I32, "int32": FHT_I32, "i64": FHT_I64, "int64": FHT_I64,
       "f32": FHT_F32, "float32": FHT_F32}
_DT_NP = {FHT_U8: np.uint8, FHT_I32: np.int32, FHT_I64: np.int64, FHT_F32: np.float32}


def _dtype_code(d) -> int:
    if isinstance(d, int):
        return d
    key = str(d).replace("torch.", "")
    if key not in _DT:
        raise InvalidArgument(f"unsupported dtype {d}")
    return _DT[key]


def _quadrant_mask(quadrants) -> int:
    if quadrants in (None, "all"):
        return 15
    if isinstance(quadrants, int):
        return quadrants
    if isinstance(quadrants, str):
        quadrants = [quadrants]
    m = 0
    for q in quadrants:
        m |= 1 << QUADRANTS.index(q)
    return m


# --------------------------------------------------------------- helpers
def split_width(w: int, strategy=SplitStrategy.Tweaked) -> tuple[int, int]:
    a, b = ctypes.c_int(), ctypes.c_int()
    check(lib().fht_split_width(w, _strategy(strategy), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def split_simple(w: int) -> tuple[int, int]:
    return split_width(w, SplitStrategy.Simple)


def split_tweaked(w: int) -> tuple[int, int]:
    return split_width(w, SplitStrategy.Tweaked)


def round_half_up_ratio(num: int, den: int) -> int:
    r = ctypes.c_int64()
    check(lib().fht_round_half_up_ratio(num, den, ctypes.byref(r)))
    return r.value


def count_additions_tree(w: int, h: int, strategy=SplitStrategy.Tweaked) -> int:
    r = ctypes.c_uint64()
    check(lib().fht_count_additions_tree(w, h, _strategy(strategy), ctypes.byref(r)))
    return int(r.value)


def rotate(v, r: int) -> np.ndarray:
    """fht::rotate (transform.cpp:8-14): u(i) = v((i + r) mod h),
    r in [0, h) or InvalidArgument.  A host helper kept for API compatibility:
    the device merge applies the same circular shift inline (its window reads
    b[(s + r) mod h], transform.cpp:53-55)."""
    a = np.asarray(v, dtype=np.int64).reshape(-1)
    h = a.size
    r = int(r)
    if r < 0 or r >= h:
        raise InvalidArgument("rotate: shift must lie in [0, h)")
    return np.concatenate((a[r:], a[:r]))


def schedule(W: int, H: int, strategy=SplitStrategy.Tweaked, block_width: int = 32, pass_levels: int = 5,
             tile_width: int = 32) -> dict:
    """The host schedule tables for one orientation (no GPU needed)."""
    need = ctypes.c_size_t()
    st = _strategy(strategy)
    lib().fht_schedule_json(W, H, st, block_width, pass_levels, tile_width, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(int(need.value) + 1)
    check(lib().fht_schedule_json(W, H, st, block_width, pass_levels, tile_width, buf, len(buf), ctypes.byref(need)))
    return json.loads(buf.value.decode())


# ----------------------------------------------- reference entry points
@dataclass
class CountedTransform:
    """transform.hpp:19-22"""
    hough: np.ndarray
    additions: int


@dataclass
class QuadrantSet:
    """quadrants.hpp:23-28"""
    horiz_pos: np.ndarray
    horiz_neg: np.ndarray
    vert_pos: np.ndarray
    vert_neg: np.ndarray


def _as_image(img) -> np.ndarray:
    a = np.asarray(img)
    if a.ndim != 2 or a.size == 0:
        raise InvalidArgument("fht2d: image is empty")
    return np.ascontiguousarray(a, dtype=np.int64)


def fht2d_counted(img, strategy=SplitStrategy.Tweaked) -> CountedTransform:
    """fht::fht2d_counted (transform.cpp:62-85) on the GPU, bit-exact int64."""
    a = _as_image(img)
    h, w = a.shape
    out = np.empty((h, w), dtype=np.int64)
    adds = ctypes.c_uint64()
    p = ctypes.POINTER(ctypes.c_int64)
    check(lib().fht_fht2d_counted_i64(a.ctypes.data_as(p), w, h, _strategy(strategy), out.ctypes.data_as(p),
                                      ctypes.byref(adds)))
    return CountedTransform(out, int(adds.value))


def fht2d(img, strategy=SplitStrategy.Tweaked) -> np.ndarray:
    """fht::fht2d (transform.cpp:87-89)."""
    return fht2d_counted(img, strategy).hough


def fht2d_quadrants(img, strategy=SplitStrategy.Tweaked, total_additions: list | None = None) -> QuadrantSet:
    """fht::fht2d_quadrants (quadrants.cpp:23-41).  If `total_additions` is a
    list, the merge-addition total is appended to it (the reference's
    optional uint64_t* out-parameter)."""
    a = _as_image(img)
    h, w = a.shape
    outs = [np.empty((h, w), np.int64), np.empty((h, w), np.int64), np.empty((w, h), np.int64),
            np.empty((w, h), np.int64)]
    adds = ctypes.c_uint64()
    p = ctypes.POINTER(ctypes.c_int64)
    check(lib().fht_fht2d_quadrants_i64(a.ctypes.data_as(p), w, h, _strategy(strategy),
                                        *[o.ctypes.data_as(p) for o in outs], ctypes.byref(adds)))
    if total_additions is not None:
        total_additions.append(int(adds.value))
    return QuadrantSet(*outs)


@dataclass
class Pattern:
    """pattern.hpp:12-17"""
    n: int
    t: int
    values: list


def fht2d_pattern(n: int, t: int, strategy=SplitStrategy.Tweaked) -> Pattern:
    """fht::fht2d_pattern (pattern.cpp:24-30, Algorithm 2)."""
    v = (ctypes.c_int * max(n, 1))()
    check(lib().fht_fht2d_pattern(n, t, _strategy(strategy), v))
    return Pattern(n, t, list(v)[:n])


def pattern_set(n: int, strategy=SplitStrategy.Tweaked) -> list:
    """fht::pattern_set (pattern.cpp:32-38)."""
    if n < 1:
        raise InvalidArgument("pattern_set: width must be positive")
    return [fht2d_pattern(n, t, strategy) for t in range(n)]


def slow_hough(img, strategy=SplitStrategy.Tweaked) -> np.ndarray:
    """fht::slow_hough (oracle.cpp:9-25): direct summation along every shifted
    pattern, on the GPU (int64, bit-exact for integer images)."""
    a = _as_image(img)
    h, w = a.shape
    out = np.empty((h, w), dtype=np.int64)
    p = ctypes.POINTER(ctypes.c_int64)
    check(lib().fht_slow_hough_i64(a.ctypes.data_as(p), w, h, _strategy(strategy), out.ctypes.data_as(p)))
    return out


def slow_hough_device(x, quadrant: str = "horiz_pos", strategy=SplitStrategy.Tweaked, stream=None):
    """Device slow_hough of one quadrant of an integer CUDA image tensor (h, w);
    returns an int64 CUDA tensor in the reference layout."""
    import torch

    if x.dim() != 2 or not x.is_cuda or not x.is_contiguous():
        raise InvalidArgument("expected a contiguous 2-D CUDA tensor")
    code = {torch.uint8: FHT_U8, torch.int32: FHT_I32, torch.int64: FHT_I64}.get(x.dtype)
    if code is None:
        raise InvalidArgument("slow_hough_device: integer images only")
    h, w = x.shape
    q = QUADRANTS.index(quadrant)
    shape = (h, w) if q < 2 else (w, h)
    out = torch.empty(shape, dtype=torch.int64, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    check(lib().fht_slow_hough_device(ctypes.c_void_p(x.data_ptr()), code, w, h, _strategy(strategy), q,
                                      ctypes.cast(ctypes.c_void_p(out.data_ptr()), ctypes.POINTER(ctypes.c_int64)),
                                      ctypes.c_void_p(st.cuda_stream)))
    return out


def check_overflow_budget(img) -> None:
    """fht::check_overflow_budget (transform.cpp:16-27), evaluated on the device."""
    import torch

    a = _as_image(img)
    t = torch.from_numpy(a).cuda()
    ok = ctypes.c_int()
    check(lib().fht_check_budget(ctypes.c_void_p(t.data_ptr()), FHT_I64, a.size, a.shape[1], ctypes.byref(ok),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


# ------------------------------------------------------------ plan API
class Plan:
    """Device-resident batched transform (fht_plan_create / fht_execute).

    Inputs: a CUDA tensor of shape (batch, h, w) or (h, w) of the plan's
    input dtype.  Outputs: a dict quadrant -> CUDA tensor (batch, H, W) in
    the reference layout (or (batch, W, H) with layout="native")."""

    def __init__(self, width: int, height: int, strategy=SplitStrategy.Tweaked, in_dtype="u8", acc_dtype="i32",
                 out_dtype=None, quadrants="all", batch: int = 1, layout: str = "reference", device: int = 0,
                 pass0_i32: bool = False):
        self.width, self.height, self.batch = int(width), int(height), int(batch)
        self.strategy = _strategy(strategy)
        self.in_dtype = _dtype_code(in_dtype)
        self.acc_dtype = _dtype_code(acc_dtype)
        self.out_dtype = self.acc_dtype if out_dtype is None else _dtype_code(out_dtype)
        self.mask = _quadrant_mask(quadrants)
        self.layout = 0 if layout == "reference" else 1
        self.device = int(device)
        h = ctypes.c_void_p()
        # pass0_i32 (acc i64): int32 sums in pass 0, for inputs with 32 * max|v| < 2^31
        acc_code = self.acc_dtype | 0x100 if pass0_i32 and self.acc_dtype == FHT_I64 else self.acc_dtype
        check(lib().fht_plan_create(self.width, self.height, self.strategy, self.in_dtype, acc_code,
                                    self.out_dtype, self.mask, self.batch, self.layout, self.device, ctypes.byref(h)))
        self._h = h
        self.workspace_bytes = int(lib().fht_workspace_bytes(h))
        self.additions = int(lib().fht_additions(h))
        self.launches = int(lib().fht_launches_per_execute(h))
        self._ws = {}
        self._ws_lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().fht_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    def describe(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 20)
        check(lib().fht_plan_describe(self._h, buf, len(buf)))
        return json.loads(buf.value.decode())

    @property
    def quadrants(self) -> list[str]:
        return [q for i, q in enumerate(QUADRANTS) if self.mask & (1 << i)]

    def out_shape(self, q: str) -> tuple[int, int]:
        horiz = q.startswith("horiz")
        W, H = (self.width, self.height) if horiz else (self.height, self.width)
        return (H, W) if self.layout == 0 else (W, H)

    def _torch_dtype(self, code):
        import torch

        return {FHT_U8: torch.uint8, FHT_I32: torch.int32, FHT_I64: torch.int64, FHT_F32: torch.float32}[code]

    def alloc_outputs(self):
        import torch

        dev = torch.device("cuda", self.device)
        return {q: torch.empty((self.batch, *self.out_shape(q)), dtype=self._torch_dtype(self.out_dtype), device=dev)
                for q in self.quadrants}

    def workspace(self, stream=None):
        """The device workspace for calls on `stream` (default: the current
        stream).  One buffer per stream: host threads may share a plan, each
        on its own stream, without sharing scratch (the reference allocates
        its scratch per call, transform.cpp:70-76)."""
        import torch

        if not self.workspace_bytes:
            return None
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        key = int(st.cuda_stream)
        with self._ws_lock:
            ws = self._ws.get(key)
            if ws is None:
                ws = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=torch.device("cuda", self.device))
                self._ws[key] = ws
        return ws

    def __call__(self, x, out: dict | None = None, stream=None):
        import torch

        if x.dim() == 2:
            x = x.unsqueeze(0)
        if tuple(x.shape) != (self.batch, self.height, self.width):
            raise InvalidArgument(f"expected input of shape {(self.batch, self.height, self.width)}, got {tuple(x.shape)}")
        if x.dtype != self._torch_dtype(self.in_dtype) or not x.is_cuda or not x.is_contiguous():
            raise InvalidArgument("input must be a contiguous CUDA tensor of the plan's input dtype")
        if out is None:
            out = self.alloc_outputs()
        ptrs = (ctypes.c_void_p * 4)()
        for i, q in enumerate(QUADRANTS):
            ptrs[i] = out[q].data_ptr() if q in out else None
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        ws = self.workspace(st)
        cells = self.width * self.height
        check(lib().fht_execute(self._h, ctypes.c_void_p(x.data_ptr()), cells, ptrs, cells,
                                ctypes.c_void_p(ws.data_ptr() if ws is not None else 0),
                                ctypes.c_void_p(st.cuda_stream)))
        return out

    def execute_host(self, x: np.ndarray, out: dict | None = None, stream=None) -> dict:
        """Host buffers in and out (fht_execute_host): H2D, transform, D2H."""
        x = np.ascontiguousarray(x)
        if x.ndim == 2:
            x = x[None]
        if x.shape != (self.batch, self.height, self.width) or x.dtype != _DT_NP[self.in_dtype]:
            raise InvalidArgument("host input has the wrong shape or dtype")
        if out is None:
            out = {q: np.empty((self.batch, *self.out_shape(q)), dtype=_DT_NP[self.out_dtype]) for q in self.quadrants}
        ptrs = (ctypes.c_void_p * 4)()
        for i, q in enumerate(QUADRANTS):
            ptrs[i] = out[q].ctypes.data if q in out else None
        st = 0
        if stream is not None:
            st = stream.cuda_stream
        check(lib().fht_execute_host(self._h, ctypes.c_void_p(x.ctypes.data), ptrs, ctypes.c_void_p(st)))
        return out

    def execute_host_ptrs(self, in_ptr: int, out_ptrs: list, stream_ptr: int = 0) -> None:
        """fht_execute_host on raw host pointers (pinned buffers from torch)."""
        ptrs = (ctypes.c_void_p * 4)(*out_ptrs)
        check(lib().fht_execute_host(self._h, ctypes.c_void_p(in_ptr), ptrs, ctypes.c_void_p(stream_ptr)))


__all__ = ["SplitStrategy", "strategy_from_string", "split_width", "split_simple", "split_tweaked",
           "round_half_up_ratio", "count_additions_tree", "rotate", "CountedTransform", "QuadrantSet", "fht2d", "Pattern",
           "fht2d_pattern", "pattern_set", "slow_hough", "slow_hough_device",
           "fht2d_counted", "fht2d_quadrants", "check_overflow_budget", "Plan", "QUADRANTS", "InvalidArgument",
           "OverflowBudget", "_lib"]
