"""CPU parity oracle for the FHT2D merge DP (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2411_07351_b200`` never imports it.

Two back ends, both plain ctypes over C/C++ shared objects built by
``oracle/Makefile``:

* ``port``  -- ``oracle/liboracle.so``: our C restatement (fht_oracle.c) of
  transform.cpp:35-85, quadrants.cpp:7-41, pattern.cpp:10-30 and
  oracle.cpp:9-33 in int64 / int32 / float32 / float64.
* ``ref``   -- ``oracle/_ref/libfhtref.so``: the unmodified reference library
  compiled from /root/reference/proj/src plus our extern "C" shim.  Present
  wherever it was built (it travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libfhtref.so"

SIMPLE, TWEAKED = 0, 1
QUADRANTS = ("horiz_pos", "horiz_neg", "vert_pos", "vert_neg")

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_u64p = ctypes.POINTER(ctypes.c_uint64)


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class OverflowBudget(OracleError, OverflowError):
    pass


def _raise(rc: int, what: str = ""):
    if rc == 0:
        return
    if rc == 1:
        raise InvalidArgument(what or "invalid argument")
    if rc == 2:
        raise OverflowBudget(what or "width * max|value| reaches 2^62")
    raise OracleError(what or f"oracle error {rc}")


def build(quiet: bool = True) -> None:
    """Compile the port and (when /root/reference exists) the reference shim."""
    import subprocess

    cmd = ["make", "-s", "-C", str(HERE)]
    subprocess.run(cmd, check=True, capture_output=quiet)


def _load(path: Path):
    if not path.exists():
        raise OracleError(f"{path} missing; run `make -C oracle`")
    return ctypes.CDLL(str(path))


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        _port = _load(PORT_SO)
        lib = _port
        for suf, ct in (("i64", ctypes.c_int64), ("i32", ctypes.c_int32), ("f32", ctypes.c_float),
                        ("f64", ctypes.c_double)):
            p = ctypes.POINTER(ct)
            f = getattr(lib, f"oracle_fht2d_{suf}")
            f.argtypes = [p, ctypes.c_int, ctypes.c_int, ctypes.c_int, p, _c_u64p]
            f.restype = ctypes.c_int
            q = getattr(lib, f"oracle_fht2d_quadrants_{suf}")
            q.argtypes = [p, ctypes.c_int, ctypes.c_int, ctypes.c_int, p, p, p, p, _c_u64p]
            q.restype = ctypes.c_int
        lib.oracle_fht2d_counted.argtypes = [_c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p, _c_u64p]
        lib.oracle_fht2d_counted.restype = ctypes.c_int
        lib.oracle_slow_hough_i64.argtypes = [_c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p]
        lib.oracle_slow_hough_i64.restype = ctypes.c_int
        lib.oracle_fht2d_pattern.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.oracle_fht2d_pattern.restype = ctypes.c_int
        lib.oracle_count_additions_tree.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.oracle_count_additions_tree.restype = ctypes.c_uint64
        lib.oracle_round_half_up_ratio.argtypes = [ctypes.c_int64, ctypes.c_int64]
        lib.oracle_round_half_up_ratio.restype = ctypes.c_int64
        lib.oracle_split_width.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int)]
        lib.oracle_split_width.restype = ctypes.c_int
        lib.oracle_batch_quadrants_u8.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p]
        lib.oracle_batch_quadrants_u8.restype = ctypes.c_int
    return _port


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        _ref = _load(REF_SO)
        lib = _ref
        cp = ctypes.c_char_p
        lib.ref_fht2d_counted.argtypes = [_c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p, _c_u64p, cp,
                                          ctypes.c_int]
        lib.ref_fht2d_quadrants.argtypes = [_c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p,
                                            _c_i64p, _c_i64p, _c_u64p, cp, ctypes.c_int]
        lib.ref_slow_hough.argtypes = [_c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p, cp, ctypes.c_int]
        lib.ref_fht2d_pattern.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), cp,
                                          ctypes.c_int]
        lib.ref_count_additions_tree.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.ref_count_additions_tree.restype = ctypes.c_uint64
        lib.ref_batch_quadrants_u8.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p, cp, ctypes.c_int]
        lib.ref_rotate.argtypes = [_c_i64p, ctypes.c_int, ctypes.c_int, _c_i64p, cp, ctypes.c_int]
        for f in ("ref_fht2d_counted", "ref_fht2d_quadrants", "ref_slow_hough", "ref_fht2d_pattern",
                  "ref_batch_quadrants_u8", "ref_rotate"):
            getattr(lib, f).restype = ctypes.c_int
    return _ref


_NP2SUF = {np.dtype(np.int64): ("i64", ctypes.c_int64), np.dtype(np.int32): ("i32", ctypes.c_int32),
           np.dtype(np.float32): ("f32", ctypes.c_float), np.dtype(np.float64): ("f64", ctypes.c_double)}


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _img(img) -> np.ndarray:
    a = np.ascontiguousarray(img)
    if a.ndim != 2:
        raise InvalidArgument("image must be 2-D (h, w) row-major")
    return a


# ---------------------------------------------------------------- port API
def fht2d(img: np.ndarray, strategy: int = TWEAKED, dtype=None):
    """Port of fht2d_counted (transform.cpp:62-85) in the element type `dtype`
    (default: int64 for integer inputs, float32/float64 kept).  `img` is (h, w)
    row-major; returns ((h, w) Hough image, J[s, t], additions)."""
    a = _img(img)
    if dtype is None:
        dtype = np.int64 if a.dtype.kind in "biu" else a.dtype
    a = np.ascontiguousarray(a, dtype=dtype)
    suf, ct = _NP2SUF[np.dtype(dtype)]
    h, w = a.shape
    out = np.empty((h, w), dtype=dtype)
    adds = ctypes.c_uint64(0)
    rc = getattr(port(), f"oracle_fht2d_{suf}")(_ptr(a, ct), w, h, strategy, _ptr(out, ct), ctypes.byref(adds))
    _raise(rc)
    return out, int(adds.value)


def fht2d_counted_i64(img: np.ndarray, strategy: int = TWEAKED):
    """Port of the reference entry point proper (int64 + overflow budget)."""
    a = np.ascontiguousarray(_img(img), dtype=np.int64)
    h, w = a.shape
    out = np.empty((h, w), dtype=np.int64)
    adds = ctypes.c_uint64(0)
    rc = port().oracle_fht2d_counted(_ptr(a, ctypes.c_int64), w, h, strategy, _ptr(out, ctypes.c_int64),
                                     ctypes.byref(adds))
    _raise(rc)
    return out, int(adds.value)


def fht2d_quadrants(img: np.ndarray, strategy: int = TWEAKED, dtype=None):
    """Port of fht2d_quadrants (quadrants.cpp:23-41).  Returns a dict of the four
    Hough images (horiz_* are (h, w), vert_* are (w, h)) and the total additions."""
    a = _img(img)
    if dtype is None:
        dtype = np.int64 if a.dtype.kind in "biu" else a.dtype
    a = np.ascontiguousarray(a, dtype=dtype)
    suf, ct = _NP2SUF[np.dtype(dtype)]
    h, w = a.shape
    outs = [np.empty((h, w), dtype=dtype), np.empty((h, w), dtype=dtype), np.empty((w, h), dtype=dtype),
            np.empty((w, h), dtype=dtype)]
    adds = ctypes.c_uint64(0)
    rc = getattr(port(), f"oracle_fht2d_quadrants_{suf}")(_ptr(a, ct), w, h, strategy, *[_ptr(o, ct) for o in outs],
                                                          ctypes.byref(adds))
    _raise(rc)
    return dict(zip(QUADRANTS, outs)), int(adds.value)


def slow_hough(img: np.ndarray, strategy: int = TWEAKED) -> np.ndarray:
    a = np.ascontiguousarray(_img(img), dtype=np.int64)
    h, w = a.shape
    out = np.empty((h, w), dtype=np.int64)
    _raise(port().oracle_slow_hough_i64(_ptr(a, ctypes.c_int64), w, h, strategy, _ptr(out, ctypes.c_int64)))
    return out


def pattern(n: int, t: int, strategy: int = TWEAKED) -> list[int]:
    v = (ctypes.c_int * max(n, 1))()
    _raise(port().oracle_fht2d_pattern(n, t, strategy, v))
    return list(v)[:n]


def count_additions_tree(w: int, h: int, strategy: int = TWEAKED) -> int:
    return int(port().oracle_count_additions_tree(w, h, strategy))


def round_half_up_ratio(num: int, den: int) -> int:
    return int(port().oracle_round_half_up_ratio(num, den))


def split_width(w: int, strategy: int = TWEAKED) -> tuple[int, int]:
    a, b = ctypes.c_int(), ctypes.c_int()
    _raise(port().oracle_split_width(w, strategy, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def batch_quadrants_u8_port(imgs: np.ndarray, strategy: int = TWEAKED, threads: int = 1, mask: int = 0xF,
                            want_output: bool = False):
    imgs = np.ascontiguousarray(imgs, dtype=np.uint8)
    n, h, w = imgs.shape
    out = np.empty((n, 4, h * w), dtype=np.int64) if want_output else None
    rc = port().oracle_batch_quadrants_u8(imgs.ctypes.data, n, w, h, strategy, mask, threads,
                                          _ptr(out, ctypes.c_int64) if out is not None else None)
    _raise(rc)
    return out


# ------------------------------------------------------------ reference API
def _err():
    return ctypes.create_string_buffer(256)


def ref_fht2d_counted(img: np.ndarray, strategy: int = TWEAKED):
    """The reference's own fht::fht2d_counted (int64)."""
    a = np.ascontiguousarray(img, dtype=np.int64)
    if a.ndim != 2:
        raise InvalidArgument("image must be 2-D")
    h, w = a.shape
    out = np.empty((h, w), dtype=np.int64)
    adds = ctypes.c_uint64(0)
    e = _err()
    rc = ref().ref_fht2d_counted(_ptr(a, ctypes.c_int64), w, h, strategy, _ptr(out, ctypes.c_int64),
                                 ctypes.byref(adds), e, 256)
    _raise(rc, e.value.decode())
    return out, int(adds.value)


def ref_fht2d_quadrants(img: np.ndarray, strategy: int = TWEAKED):
    a = np.ascontiguousarray(img, dtype=np.int64)
    h, w = a.shape
    outs = [np.empty((h, w), np.int64), np.empty((h, w), np.int64), np.empty((w, h), np.int64),
            np.empty((w, h), np.int64)]
    adds = ctypes.c_uint64(0)
    e = _err()
    rc = ref().ref_fht2d_quadrants(_ptr(a, ctypes.c_int64), w, h, strategy,
                                   *[_ptr(o, ctypes.c_int64) for o in outs], ctypes.byref(adds), e, 256)
    _raise(rc, e.value.decode())
    return dict(zip(QUADRANTS, outs)), int(adds.value)


def ref_rotate(v, r: int) -> np.ndarray:
    """The reference's own fht::rotate (transform.cpp:8-14)."""
    a = np.ascontiguousarray(v, dtype=np.int64).reshape(-1)
    out = np.empty_like(a)
    e = _err()
    _raise(ref().ref_rotate(_ptr(a, ctypes.c_int64), a.size, int(r), _ptr(out, ctypes.c_int64), e, 256),
           e.value.decode())
    return out


def ref_slow_hough(img: np.ndarray, strategy: int = TWEAKED) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.int64)
    h, w = a.shape
    out = np.empty((h, w), np.int64)
    e = _err()
    _raise(ref().ref_slow_hough(_ptr(a, ctypes.c_int64), w, h, strategy, _ptr(out, ctypes.c_int64), e, 256),
           e.value.decode())
    return out


def ref_pattern(n: int, t: int, strategy: int = TWEAKED) -> list[int]:
    v = (ctypes.c_int * max(n, 1))()
    e = _err()
    _raise(ref().ref_fht2d_pattern(n, t, strategy, v, e, 256), e.value.decode())
    return list(v)[:n]


def ref_count_additions_tree(w: int, h: int, strategy: int = TWEAKED) -> int:
    return int(ref().ref_count_additions_tree(w, h, strategy))


def ref_batch_quadrants_u8(imgs: np.ndarray, strategy: int = TWEAKED, threads: int = 1, mask: int = 0xF,
                           want_output: bool = False):
    imgs = np.ascontiguousarray(imgs, dtype=np.uint8)
    n, h, w = imgs.shape
    out = np.empty((n, 4, h * w), dtype=np.int64) if want_output else None
    e = _err()
    rc = ref().ref_batch_quadrants_u8(imgs.ctypes.data, n, w, h, strategy, mask, threads,
                                      _ptr(out, ctypes.c_int64) if out is not None else None, e, 256)
    _raise(rc, e.value.decode())
    return out


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
