"""ctypes binding of libtqr.so (the C ABI declared in include/tqr.h).

The library is built in-tree by ``paper_1303_3182_b200/_build.py`` (called
from ``__graft_entry__.build()``).  There is no fallback: if the shared
library is missing the import of the engine fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TQR_LIB_PATH: an instrumented build (tools/, profiling only)
LIB_PATH = os.environ.get("TQR_LIB_PATH") or os.path.join(HERE, "libtqr.so")

TQR_OK, TQR_EVALUE, TQR_EKEY, TQR_EASSERT, TQR_EOTHER, TQR_ECUDA = 0, -1, -2, -3, -4, -5
TQR_NO_BS = -(2 ** 31)

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
i8p = C.POINTER(C.c_int8)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class BuildInfo(C.Structure):
    _fields_ = [("p", C.c_int32), ("q", C.c_int32), ("family_ts", C.c_int32),
                ("cp", C.c_int64), ("total_weight", C.c_int64),
                ("counts", C.c_int64 * 6),
                ("n_elim", C.c_int64), ("n_trace", C.c_int64),
                ("n_zeroed", C.c_int64), ("n_updates", C.c_int64)]


class PlanInfo(C.Structure):
    _fields_ = [("p", C.c_int32), ("q", C.c_int32), ("nb", C.c_int32), ("ib", C.c_int32),
                ("slab", C.c_int32), ("family_ts", C.c_int32),
                ("n_tasks", C.c_int64), ("n_items", C.c_int64), ("n_preds", C.c_int64),
                ("tg_stride", C.c_int64), ("te_stride", C.c_int64),
                ("flops_alg", C.c_double)]


# name -> (restype, argtypes); must list every symbol include/tqr.h declares
SIGNATURES = {
    "tqr_last_error": (C.c_char_p, []),
    "tqr_abi_version": (C.c_int, []),
    "tqr_coarse_schedule": (C.c_int, [C.c_int, C.c_int, C.c_char_p, i32p, i32p, C.c_int64, i64p, i32p]),
    "tqr_plasmatree_list": (C.c_int, [C.c_int, C.c_int, C.c_int, i32p, C.c_int64, i64p]),
    "tqr_elim_validate": (C.c_int, [C.c_int, C.c_int, i32p, C.c_int64, C.c_char_p, C.c_int64]),
    "tqr_elim_with_steps": (C.c_int, [i32p, C.c_int64, i32p]),
    "tqr_elim_normalized": (C.c_int, [C.c_int, C.c_int, i32p, C.c_int64, i32p]),
    "tqr_build_tree": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int, i64p,
                                 C.c_int, C.c_int, C.POINTER(vp)]),
    "tqr_tiled_build": (C.c_int, [C.c_int, C.c_int, i32p, C.c_int64, C.c_int, i64p, C.c_int, C.c_int,
                                  C.c_int, C.POINTER(vp)]),
    "tqr_build_get_info": (C.c_int, [vp, C.POINTER(BuildInfo)]),
    "tqr_build_get_elim": (C.c_int, [vp, i32p]),
    "tqr_build_get_zeroed": (C.c_int, [vp, i64p]),
    "tqr_build_get_trace": (C.c_int, [vp, i8p, i32p, i64p]),
    "tqr_build_get_updates": (C.c_int, [vp, i64p]),
    "tqr_build_hazard_edges": (C.c_int, [vp, i32p, C.c_int64, i64p]),
    "tqr_trace_build": (C.c_int, [C.c_int, C.c_int, i8p, i32p, C.c_int64, C.POINTER(vp)]),
    "tqr_build_free": (None, [vp]),
    "tqr_plan_create": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    "tqr_plan_create_io": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "tqr_plan_get_info": (C.c_int, [vp, C.POINTER(PlanInfo)]),
    "tqr_plan_free": (None, [vp]),
    "tqr_pack": (C.c_int, [vp, C.c_int64, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp]),
    "tqr_unpack": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int64, C.c_int, vp]),
    "tqr_extract_r": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int64, C.c_int, vp]),
    "tqr_factor": (C.c_int, [vp, vp, vp, vp, vp]),
    "tqr_factor_io": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, C.c_int64, vp, vp]),
    "tqr_qr_host": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "tqr_plan_arrival_units": (C.c_int, [vp, i32p, i32p]),
    "tqr_apply_q": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, C.c_int, vp]),
    "tqr_fp64_peak": (C.c_int, [f64p, vp]),
    "tqr_set_trace": (C.c_int, [vp]),
    "tqr_plan_items": (C.c_int, [vp, i32p]),
}

_lib = None


def lib():
    """Load libtqr.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the engine first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        missing = [n for n in SIGNATURES if not hasattr(L, n)]
        if missing:
            raise ImportError(f"{LIB_PATH} lacks symbols {missing}: rebuild it")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    """Raise the Python exception class matching a TQR_E* status."""
    if rc == TQR_OK:
        return
    msg = lib().tqr_last_error().decode()
    if rc == TQR_EVALUE:
        raise ValueError(msg)
    if rc == TQR_EKEY:
        raise KeyError(msg)
    if rc == TQR_EASSERT:
        raise AssertionError(msg)
    raise RuntimeError(f"libtqr status {rc}: {msg}")


def as_i32(arr):
    a = np.ascontiguousarray(arr, dtype=np.int32)
    return a, a.ctypes.data_as(i32p)


def ptr_i32(a):
    return a.ctypes.data_as(i32p)


def ptr_i64(a):
    return a.ctypes.data_as(i64p)
