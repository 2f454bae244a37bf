"""ctypes binding of the C ABI in include/fht_b200.h (libfht_b200.so).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libfht_b200.so"

FHT_OK, FHT_ERR_INVALID, FHT_ERR_OVERFLOW, FHT_ERR_CUDA, FHT_ERR_NOMEM, FHT_ERR_INTERNAL = range(6)
FHT_U8, FHT_I32, FHT_I64, FHT_F32 = range(4)
FHT_HORIZ_POS, FHT_HORIZ_NEG, FHT_VERT_POS, FHT_VERT_NEG = 1, 2, 4, 8
FHT_ALL_QUADRANTS = 15
FHT_LAYOUT_REFERENCE, FHT_LAYOUT_NATIVE = 0, 1

# Every symbol include/fht_b200.h declares: (name, restype, argtypes).
_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_pi = ctypes.POINTER(ctypes.c_int)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pu64 = ctypes.POINTER(ctypes.c_uint64)
SIGNATURES = {
    "fht_plan_create": (_i, [_i, _i, _i, _i, _i, _i, _i, _i, _i, _i, ctypes.POINTER(_vp)]),
    "fht_plan_destroy": (_i, [_vp]),
    "fht_workspace_bytes": (ctypes.c_size_t, [_vp]),
    "fht_additions": (_u64, [_vp]),
    "fht_launches_per_execute": (_i, [_vp]),
    "fht_plan_describe": (_i, [_vp, ctypes.c_char_p, ctypes.c_size_t]),
    "fht_execute": (_i, [_vp, _vp, _i64, ctypes.POINTER(_vp), _i64, _vp, _vp]),
    "fht_execute_host": (_i, [_vp, _vp, ctypes.POINTER(_vp), _vp]),
    "fht_execute_pitched": (_i, [_vp, _vp, _i64, _i64, ctypes.POINTER(_vp), _i64, _vp, _vp]),
    "fht_merge_root": (_i, [_i, _i, _i, _i, _i, _i, _vp, _i, _vp, _i, _i, _i, _vp, _vp]),
    "fht_execute_pitched_peer": (_i, [_vp, _vp, _i64, ctypes.POINTER(_vp), _vp, _vp, _i, _i, _vp]),
    "fht_ipc_get_handle": (_i, [_vp, _vp, ctypes.c_size_t]),
    "fht_ipc_open_handle": (_i, [_vp, ctypes.c_size_t, _i, ctypes.POINTER(_vp)]),
    "fht_ipc_close": (_i, [_vp]),
    "fht_device_alloc": (_i, [ctypes.c_size_t, _i, ctypes.POINTER(_vp)]),
    "fht_device_free": (_i, [_vp]),
    "fht_execute_profiled": (_i, [_vp, _vp, _i64, ctypes.POINTER(_vp), _i64, _vp, _vp, ctypes.POINTER(ctypes.c_float),
                                  _pi, ctypes.POINTER(ctypes.c_double), _i, _pi]),
    "fht_check_budget": (_i, [_vp, _i, _i64, _i, _pi, _vp]),
    "fht_fht2d_counted_i64": (_i, [_pi64, _i, _i, _i, _pi64, _pu64]),
    "fht_fht2d_quadrants_i64": (_i, [_pi64, _i, _i, _i, _pi64, _pi64, _pi64, _pi64, _pu64]),
    "fht_slow_hough_device": (_i, [_vp, _i, _i, _i, _i, _i, _pi64, _vp]),
    "fht_slow_hough_i64": (_i, [_pi64, _i, _i, _i, _pi64]),
    "fht_fht2d_pattern": (_i, [_i, _i, _i, _pi]),
    "fht_max_deviation_numerators": (_i, [_i, _i, _i, _pi64]),
    "fht_split_width": (_i, [_i, _i, _pi, _pi]),
    "fht_round_half_up_ratio": (_i, [_i64, _i64, _pi64]),
    "fht_count_additions_tree": (_i, [_i, _i, _i, _pu64]),
    "fht_schedule_json": (_i, [_i, _i, _i, _i, _i, _i, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "fht_plan_cache_clear": (_i, [ctypes.POINTER(ctypes.c_size_t)]),
    "fht_plan_cache_size": (ctypes.c_size_t, []),
    "fht_debug_counters": (_i, [_pu64, _pu64]),
    "fht_last_error": (ctypes.c_char_p, []),
    "fht_version": (ctypes.c_char_p, []),
}


class FhtError(RuntimeError):
    """Base class; the subclasses mirror the reference's exception types."""


class InvalidArgument(FhtError, ValueError):
    """std::invalid_argument in the reference (transform.cpp:63, split.hpp:34,41,54-55)."""


class OverflowBudget(FhtError, OverflowError):
    """std::overflow_error in the reference (transform.cpp:24-26)."""


class CudaError(FhtError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        l = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def debug_counters() -> tuple[int, int]:
    """(stream synchronisations, device allocations) the library has made so far."""
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib().fht_debug_counters(ctypes.byref(a), ctypes.byref(b)))
    return int(a.value), int(b.value)


def check(rc: int) -> None:
    if rc == FHT_OK:
        return
    msg = (lib().fht_last_error() or b"").decode()
    if rc == FHT_ERR_INVALID:
        raise InvalidArgument(msg)
    if rc == FHT_ERR_OVERFLOW:
        raise OverflowBudget(msg)
    if rc == FHT_ERR_CUDA:
        raise CudaError(msg)
    if rc == FHT_ERR_NOMEM:
        raise MemoryError(msg)
    raise FhtError(f"fht error {rc}: {msg}")


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def env_flag(name: str, default: str = "") -> str:
    return os.environ.get(name, default)
