"""ctypes loader for the in-tree CUDA library (argument marshalling only).

There is no fallback: if libaim_b200.so is missing or cannot be loaded the
import fails loudly (build it with `python -c "import __graft_entry__ as g; g.build()"`).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AIM_LIB") or os.path.join(HERE, "libaim_b200.so")


class AimInfo(ctypes.Structure):
    _fields_ = [
        ("n_rwg", ctypes.c_int64), ("n_tri", ctypes.c_int64),
        ("M", ctypes.c_int32), ("S", ctypes.c_int32),
        ("grid_origin", ctypes.c_int32 * 3), ("grid_dims", ctypes.c_int32 * 3), ("fft_dims", ctypes.c_int32 * 3),
        ("n_nodes", ctypes.c_int64), ("nnz_proj", ctypes.c_int64), ("nnz_near", ctypes.c_int64),
        ("k", ctypes.c_double), ("h", ctypes.c_double), ("near_radius", ctypes.c_double),
        ("device_bytes", ctypes.c_int64), ("plan_seconds", ctypes.c_double),
        ("conv_mode", ctypes.c_int32), ("precision", ctypes.c_int32),
    ]


# (name, restype, argtypes) for every symbol declared in include/aim.h
P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
D = ctypes.c_double
SIGNATURES = [
    ("aim_plan_create", I32, [P, I64, P, I64, P, I64, D, D, I32, D, I32, P, ctypes.POINTER(P)]),
    ("aim_plan_destroy", I32, [P]),
    ("aim_plan_info", I32, [P, ctypes.POINTER(AimInfo)]),
    ("aim_matvec", I32, [P, P, P, I32, P]),
    ("aim_matvec_host", I32, [P, P, P, I32]),
    ("aim_matvec_host_steps", I32, [P, P, P, I32, I32]),
    ("aim_gmres", I32, [P, P, P, I32, D, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(D)]),
    ("aim_gmres_history", I32, [P, P, I32, ctypes.POINTER(I32)]),
    ("aim_precond_build", I32, [P, I32]),
    ("aim_precond_apply", I32, [P, P, P, P]),
    ("aim_precond_info", I32, [P, P]),
    ("aim_plan_compress", I32, [P, I32]),
    ("aim_compress_info", I32, [P, P]),
    ("aim_plan_elements", I32, [P, P, P, ctypes.POINTER(I32)]),
    ("aim_reduced_set", I32, [P, I32, P, P, P, P, P, P, P, I32]),
    ("aim_reduced_matvec", I32, [P, P, P, P]),
    ("aim_reduced_gmres", I32, [P, P, P, I32, D, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(D)]),
    ("aim_planewave_rhs", I32, [P, P, P, D, D, P, P]),
    ("aim_project", I32, [P, P, P, I32, P]),
    ("aim_convolve", I32, [P, P, P, I32, P]),
    ("aim_interpolate", I32, [P, P, P, P, I32, I32, P]),
    ("aim_plan_export", I32, [P, I32, P, I64]),
    ("aim_profile", I32, [P, I32]),
    ("aim_profile_read", I32, [P, ctypes.POINTER(D), ctypes.POINTER(I64)]),
    ("aim_slab_partition", I32, [P, I64, P, I64, P, I64, D, I32, I32, P, P, P]),
    ("aim_nccl_unique_id", I32, [P, I64]),
    ("aim_slab_create", I32, [P, I64, P, I64, P, I64, D, D, I32, D, I32, I32, P, ctypes.POINTER(P)]),
    ("aim_slab_matvec", I32, [P, P, P, I32, P]),
    ("aim_slab_gmres", I32, [P, P, P, I32, D, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(D)]),
    ("aim_slab_query", I32, [P, I32, P]),
    ("aim_slab_destroy", I32, [P]),
    ("aim_last_error", ctypes.c_char_p, []),
    ("aim_launch_count", I64, [I32]),
]

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib
