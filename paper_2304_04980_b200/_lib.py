"""ctypes binding of libgridlq_b200.so (declarations in include/gridlq_b200.h).

The library is built in-tree (``paper_2304_04980_b200/build.py``).  There is no CPU
fallback: if the shared object is missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (BreakdownError, DimensionMismatchError, GridLQError, MaxIterationsExceeded,
                     NotPositiveDefiniteError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgridlq_b200.so")

GQ_OK, GQ_MAX_ITER, GQ_BREAKDOWN, GQ_DIM_MISMATCH, GQ_INVALID_ARG, GQ_NOT_SPD, \
    GQ_CUDA_ERROR, GQ_UNSUPPORTED = range(8)
GQ_VEC_X, GQ_VEC_R = 0, 1
# stage-slab mode (include/gridlq_b200.h)
GQ_SLAB_INIT_OUTER, GQ_SLAB_INIT_FINISH, GQ_SLAB_DELTA, GQ_SLAB_UPDATE, GQ_SLAB_OUTER, \
    GQ_SLAB_DIRECTION = range(6)
GQ_SLAB_VEC_D, GQ_SLAB_VEC_DL0, GQ_SLAB_VEC_DL1 = range(3)
GQ_SLAB_CURV, GQ_SLAB_RES, GQ_SLAB_MU = range(3)

EXPORTS = (
    "gq_last_error", "gq_version", "gq_create", "gq_destroy", "gq_dim", "gq_set_stream",
    "gq_synchronize", "gq_set_sweeps", "gq_apply_delta", "gq_apply_outer_coupling",
    "gq_apply_inner_coupling", "gq_pair_solve", "gq_apply_precond", "gq_pcg_start",
    "gq_pcg_run", "gq_pcg_read", "gq_pcg_history", "gq_pcg_scalars", "gq_pcg",
    "gq_profile_steps", "gq_kernel_name", "gq_launches_per_step", "gq_input_dim",
    "gq_recover", "gq_kkt_residual", "gq_nbjm_solve", "gq_slab_enable", "gq_slab_start",
    "gq_slab_phase", "gq_slab_pack", "gq_slab_unpack", "gq_slab_scalar_ptr", "gq_slab_status",
    "gq_build_offset", "gq_touch_pages", "gq_host_alloc", "gq_host_free",
)


class GqProblemDesc(ctypes.Structure):
    _fields_ = [
        ("K", ctypes.c_int32), ("N", ctypes.c_int32), ("T", ctypes.c_int32),
        ("n", ctypes.c_int32), ("m", ctypes.c_int32),
        ("n_dyn", ctypes.c_int32), ("n_cost", ctypes.c_int32),
        ("dyn_class", ctypes.POINTER(ctypes.c_int32)),
        ("cost_class", ctypes.POINTER(ctypes.c_int32)),
        ("A", ctypes.POINTER(ctypes.c_double)), ("B", ctypes.POINTER(ctypes.c_double)),
        ("R", ctypes.POINTER(ctypes.c_double)), ("C", ctypes.POINTER(ctypes.c_double)),
        ("Q", ctypes.POINTER(ctypes.c_double)),
    ]


_lib = None


def load():
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is not built; run `python -m paper_2304_04980_b200.build` "
            "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, dp, i32, i64 = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "gq_last_error": (ctypes.c_char_p, []),
        "gq_version": (ctypes.c_char_p, []),
        "gq_create": (ctypes.c_int, [ctypes.POINTER(GqProblemDesc), i32, i32,
                                     ctypes.POINTER(ctypes.c_void_p)]),
        "gq_destroy": (None, [vp]),
        "gq_dim": (i64, [vp]),
        "gq_set_stream": (ctypes.c_int, [vp, vp]),
        "gq_synchronize": (ctypes.c_int, [vp]),
        "gq_set_sweeps": (ctypes.c_int, [vp, i32, i32]),
        "gq_apply_delta": (ctypes.c_int, [vp, dp, dp]),
        "gq_apply_outer_coupling": (ctypes.c_int, [vp, dp, dp]),
        "gq_apply_inner_coupling": (ctypes.c_int, [vp, dp, dp]),
        "gq_pair_solve": (ctypes.c_int, [vp, dp, dp]),
        "gq_apply_precond": (ctypes.c_int, [vp, dp, dp]),
        "gq_pcg_start": (ctypes.c_int, [vp, dp, dp, i32]),
        "gq_pcg_run": (ctypes.c_int, [vp, ctypes.c_double, i64, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int32)]),
        "gq_pcg_read": (ctypes.c_int, [vp, i32, dp]),
        "gq_pcg_history": (ctypes.c_int, [vp, dp, i64]),
        "gq_pcg_scalars": (ctypes.c_int, [vp] + [ctypes.POINTER(ctypes.c_double)] * 4),
        "gq_pcg": (ctypes.c_int, [vp, dp, dp, ctypes.c_double, i64, i32, dp, dp, i64,
                                  ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)]),
        "gq_profile_steps": (ctypes.c_int, [vp, i32, ctypes.POINTER(ctypes.c_float), i32]),
        "gq_kernel_name": (ctypes.c_char_p, [vp, i32]),
        "gq_launches_per_step": (ctypes.c_int, [vp]),
        "gq_input_dim": (i64, [vp]),
        "gq_recover": (ctypes.c_int, [vp, dp, dp, dp, ctypes.POINTER(ctypes.c_double)]),
        "gq_kkt_residual": (ctypes.c_int, [vp, dp, dp, dp, dp, dp]),
        "gq_nbjm_solve": (ctypes.c_int, [vp, dp, ctypes.c_double, i64, dp,
                                         ctypes.POINTER(ctypes.c_int64)]),
        "gq_slab_enable": (ctypes.c_int, [vp, i32, i32]),
        "gq_slab_start": (ctypes.c_int, [vp, dp, dp, i32, ctypes.c_double, i64]),
        "gq_slab_phase": (ctypes.c_int, [vp, i32, i32]),
        "gq_slab_pack": (ctypes.c_int, [vp, i32, i32, dp]),
        "gq_slab_unpack": (ctypes.c_int, [vp, i32, i32, dp]),
        "gq_slab_scalar_ptr": (ctypes.c_void_p, [vp, i32]),
        "gq_slab_status": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_int64)]
                           + [ctypes.POINTER(ctypes.c_int32)] * 3),
        "gq_build_offset": (ctypes.c_int, [i32, i32, i32, i32, i32, dp, dp, dp, dp, dp, vp]),
        "gq_touch_pages": (None, [vp, i64]),
        "gq_host_alloc": (ctypes.c_void_p, [i64]),
        "gq_host_free": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().gq_last_error().decode()


def check(rc: int, what: str = ""):
    """Map a gq_status onto the gridlq exception types (MAX_ITER / BREAKDOWN are left to
    the caller, which owns the iterate and report)."""
    if rc == GQ_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == GQ_DIM_MISMATCH:
        raise DimensionMismatchError(msg)
    if rc == GQ_INVALID_ARG:
        raise ValueError(msg)
    if rc == GQ_NOT_SPD:
        raise NotPositiveDefiniteError(msg)
    if rc == GQ_BREAKDOWN:
        raise BreakdownError(msg)
    if rc == GQ_MAX_ITER:
        raise MaxIterationsExceeded(msg)
    if rc == GQ_UNSUPPORTED:
        raise DimensionMismatchError(msg)
    raise GridLQError(f"CUDA error: {msg}")
