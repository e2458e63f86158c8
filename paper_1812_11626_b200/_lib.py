"""ctypes loader for libsunfold.so and the C structs of include/sunfold.h."""
from __future__ import annotations

import ctypes
import os
import re

from . import _build

_lib = None

P = ctypes.c_void_p


class SunZCSR(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz", ctypes.c_int64), ("row_ptr", P), ("col", P), ("val", P)]


class SunDCSR(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", P), ("col", P), ("val", P)]


class SunPlanInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("P", ctypes.c_int32),
        ("w_h0", ctypes.c_int32), ("w_h1", ctypes.c_int32), ("w_l", ctypes.c_int32), ("w_k", ctypes.c_int32),
        ("tau_q0", ctypes.c_double), ("tau_q1", ctypes.c_double),
        ("mode_q0", ctypes.c_int32), ("mode_q1", ctypes.c_int32),
        ("pairs_per_tile_q0", ctypes.c_int32), ("pairs_per_tile_q1", ctypes.c_int32),
        ("tiles_q0", ctypes.c_int64), ("tiles_q1", ctypes.c_int64),
        ("has_h1", ctypes.c_int32),
        ("npos_far_q0", ctypes.c_int32), ("npos_far_q1", ctypes.c_int32),
        ("launches_count", ctypes.c_int32), ("launches_fill", ctypes.c_int32),
    ]


SIGNATURES = {
    "sun_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "sun_workspace_bytes_ops": (ctypes.c_size_t, [P, P, P, ctypes.c_int32]),
    "sun_plan_create": (ctypes.c_int, [P, P, P, P, P, ctypes.c_int32, P, ctypes.c_size_t, P]),
    "sun_plan_create_ex": (ctypes.c_int, [P, P, P, P, P, ctypes.c_int32, ctypes.c_int32, P, ctypes.c_size_t, P]),
    "sun_count": (ctypes.c_int, [P, P]),
    "sun_plan_nnz": (ctypes.c_int, [P, P, P]),
    "sun_unfold": (ctypes.c_int, [P, P, P, P, P]),
    "sun_apply": (ctypes.c_int, [P, P, ctypes.c_double, P, P, P, P]),
    "sun_run": (ctypes.c_int, [P, P, P, P, P]),
    "sun_nnz_bound": (ctypes.c_int64, [P, ctypes.c_int32]),
    "sun_plan_info": (ctypes.c_int, [P, P]),
    "sun_plan_set_graphs": (ctypes.c_int, [P, ctypes.c_int32]),
    "sun_plan_stash_bytes": (ctypes.c_size_t, [P]),
    "sun_plan_set_stash": (ctypes.c_int, [P, P, ctypes.c_size_t]),
    "sun_plan_set_timing": (ctypes.c_int, [P, ctypes.c_int32]),
    "sun_plan_phase_ms": (ctypes.c_int, [P, P, P]),
    "sun_expand_state": (ctypes.c_int, [P, P, P]),
    "sun_state_diag": (ctypes.c_int, [P, ctypes.c_int32, P, P]),
    "sun_rk4": (ctypes.c_int, [P, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int64, P, P, P]),
    "sun_rk4_work_bytes": (ctypes.c_size_t, [ctypes.c_int64]),
    "sun_rk4_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_void_p]),
    "sun_rk4_plan_work_bytes": (ctypes.c_size_t, [ctypes.c_void_p]),
    "sun_apply_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_size_t, ctypes.c_void_p]),
    "sun_structure_constants": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.c_void_p]),
    "sun_sc_work_bytes": (ctypes.c_size_t, [ctypes.c_int32]),
    "sun_state_reconstruct": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "sun_unfold_dense": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p]),
    "sun_dense_work_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "sun_dense_launches": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_size_t]),
    "sun_plan_destroy": (None, [P]),
    "sun_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "sun_gen_index": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "sun_version": (ctypes.c_char_p, []),
}


def header_symbols() -> list:
    """Function names declared in include/sunfold.h (the ABI the .so must export)."""
    src = open(os.path.join(_build.ROOT, "include", "sunfold.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sun_[a-z_0-9]+)\s*\(", src)))


def load():
    """Load (building first if needed) the in-tree libsunfold.so.  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SUNFOLD_LIB") or _build.LIB  # SUNFOLD_LIB: diagnostics builds only
    if path == _build.LIB and _build.stale():
        try:
            _build.build()
        except Exception as e:  # no fallback: the product path needs the CUDA library
            raise RuntimeError(f"libsunfold.so is missing/stale and could not be built: {e}") from e
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
