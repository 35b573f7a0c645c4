"""ctypes binding of the C ABI in include/b200sort.h (libb200sort.so).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) into
``paper_1105_6040_b200/lib``. There is no fallback: if the shared object is
missing or no sm_100 device is present, loading / context creation raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B2S_LIB") or os.path.join(HERE, "lib", "libb200sort.so")

B2S_OK, B2S_EINVAL, B2S_ENOMEM, B2S_ECUDA, B2S_EINTERNAL, B2S_ENCCL = range(6)
B2S_XCHG_AUTO, B2S_XCHG_P2P, B2S_XCHG_NCCL = range(3)
B2S_I32, B2S_U32, B2S_I64, B2S_U64 = range(4)
B2S_DEVICE, B2S_HOST = 0, 1

# every symbol include/b200sort.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "b2s_create", "b2s_destroy", "b2s_set_stream", "b2s_synchronize", "b2s_enable_timing",
    "b2s_get_timing", "b2s_last_error", "b2s_version", "b2s_device_count", "b2s_kernel_launches", "b2s_lane_ordered_atomics", "b2s_sort",
    "b2s_merge", "b2s_sort_batch", "b2s_partitioned_sort", "b2s_odd_even_sort", "b2s_plan_partition",
    "b2s_merge_split_padded",
    "b2s_sample_regular", "b2s_select_splitters", "b2s_bucket_bounds", "b2s_gen_keys",
    "b2s_check_sorted", "b2s_gen_zipf", "b2s_exchange_buffer", "b2s_open_peer", "b2s_close_peers",
    "b2s_create_multi", "b2s_destroy_multi", "b2s_multi_info", "b2s_multi_set_transport",
    "b2s_multi_get_timing", "b2s_sample_sort",
]


class b2s_timing(ctypes.Structure):
    _fields_ = [
        ("hist_ms", ctypes.c_float),
        ("pass_ms", ctypes.c_float * 8),
        ("passes_executed", ctypes.c_int),
        ("passes_possible", ctypes.c_int),
        ("copy_ms", ctypes.c_float),
        ("merge_ms", ctypes.c_float),
        ("merge_rounds", ctypes.c_int),
        ("total_ms", ctypes.c_float),
    ]


class b2s_multi_timing(ctypes.Structure):
    _fields_ = [
        ("local_sort_ms", ctypes.c_float),
        ("splitters_ms", ctypes.c_float),
        ("exchange_merge_ms", ctypes.c_float),
        ("total_ms", ctypes.c_float),
        ("transport", ctypes.c_int),
        ("max_bucket", ctypes.c_uint64),
        ("min_bucket", ctypes.c_uint64),
    ]


class b2s_sample(ctypes.Structure):
    _fields_ = [("key", ctypes.c_uint64), ("tag", ctypes.c_uint64)]


_p = ctypes.c_void_p
_u64 = ctypes.c_uint64
_i = ctypes.c_int
_u32 = ctypes.c_uint32
_st = ctypes.c_int

_SIGS = {
    "b2s_create": (_st, [_i, ctypes.POINTER(_p)]),
    "b2s_destroy": (_st, [_p]),
    "b2s_set_stream": (_st, [_p, _p]),
    "b2s_synchronize": (_st, [_p]),
    "b2s_enable_timing": (_st, [_p, _i]),
    "b2s_get_timing": (_st, [_p, ctypes.POINTER(b2s_timing)]),
    "b2s_last_error": (ctypes.c_char_p, []),
    "b2s_version": (ctypes.c_char_p, []),
    "b2s_device_count": (_i, []),
    "b2s_kernel_launches": (ctypes.c_ulonglong, []),
    "b2s_lane_ordered_atomics": (_i, [_p]),
    "b2s_sort": (_st, [_p, _i, _p, _p, _p, _p, _u64, _u32]),
    "b2s_merge": (_st, [_p, _i, _p, _p, _p, _i, _p, _p, _u32]),
    "b2s_sort_batch": (_st, [_p, _i, _p, _p, _p, _p, _u64, _i, _u32]),
    "b2s_partitioned_sort": (_st, [_p, _i, _p, _p, _p, _p, _u64, _i, _u32]),
    "b2s_odd_even_sort": (_st, [_p, _i, _p, _p, _u64, _i, _u32]),
    "b2s_plan_partition": (_st, [_u64, _i, _p]),
    "b2s_merge_split_padded": (_st, [_p, _i, _p, _u64, _u64, _p, _u64, _u64, _i, _p, _p, _p,
                                     _u32]),
    "b2s_sample_regular": (_st, [_p, _i, _p, _u64, _i, _i, _p]),
    "b2s_select_splitters": (_st, [_p, _p, _i, _i, _p]),
    "b2s_bucket_bounds": (_st, [_p, _i, _p, _u64, _i, _p, _i, _p]),
    "b2s_gen_keys": (_st, [_p, _i, _u64, _u64, _u64, _i, _p, _u32]),
    "b2s_check_sorted": (_st, [_p, _i, _p, _u64, _p, _p, _p, _u32]),
    "b2s_gen_zipf": (_st, [_p, _i, _u64, _u64, _u64, _p, _u32, _p, _u32]),
    "b2s_exchange_buffer": (_st, [_p, _u64, ctypes.POINTER(_p), _p]),
    "b2s_open_peer": (_st, [_p, _p, ctypes.POINTER(_p)]),
    "b2s_close_peers": (_st, [_p]),
    "b2s_create_multi": (_st, [_i, _p, ctypes.POINTER(_p)]),
    "b2s_destroy_multi": (_st, [_p]),
    "b2s_multi_info": (_st, [_p, _p, _p, _p, _p]),
    "b2s_multi_set_transport": (_st, [_p, _i]),
    "b2s_multi_get_timing": (_st, [_p, ctypes.POINTER(b2s_multi_timing)]),
    "b2s_sample_sort": (_st, [_p, _i, _p, _p, _p, _p, _p, _p, _p, _i, _u32]),
}


class B2SError(RuntimeError):
    """A non-OK b2s_status. ``status`` holds the code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Loads libb200sort.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`). "
                "There is no CPU fallback.")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(status: int) -> None:
    if status != B2S_OK:
        from . import errors
        msg = lib().b2s_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)
