"""ctypes binding of include/diffpd_b200.h (argument marshalling only).

Every computation happens in libdiffpd_b200.so (sm_100a kernels + host setup).
There is no CPU fallback: loading fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdiffpd_b200.so")

PD_OK, PD_ERR_INVALID_ARGUMENT, PD_ERR_NUMERICAL, PD_ERR_CUDA, PD_ERR_STATE = range(5)
STATUS_NAMES = {0: "PD_OK", 1: "PD_ERR_INVALID_ARGUMENT", 2: "PD_ERR_NUMERICAL", 3: "PD_ERR_CUDA",
                4: "PD_ERR_STATE"}

# every symbol include/diffpd_b200.h declares
EXPORTS = ["pd_create", "pd_forward", "pd_backward", "pd_backward_steps", "pd_eval_objective", "pd_apply_Ainv", "pd_apply_AN",
           "pd_project_rotations", "pd_polar_stats", "pd_info", "pd_profile", "pd_contact_sets", "pd_last_error",
           "pd_destroy"]

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)


class PdMesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_elems", C.c_int32), ("rest_xyz", dp), ("hex8", ip),
                ("dx", C.c_double)]


class PdMaterial(C.Structure):
    _fields_ = [("youngs", C.c_double), ("poisson", C.c_double), ("density", C.c_double),
                ("muscle_w", C.c_double), ("gravity", C.c_double * 3), ("fiber", C.c_double * 3),
                ("volume", C.c_int32), ("fiber_dir", dp)]


class PdOptions(C.Structure):
    _fields_ = [("tol_fwd", C.c_double), ("tol_adj", C.c_double), ("max_iter_fwd", C.c_int32),
                ("max_iter_adj", C.c_int32), ("fixed_iter", C.c_int32), ("accel_fwd", C.c_int32),
                ("accel_adj", C.c_int32), ("check_every", C.c_int32), ("max_batch", C.c_int32),
                ("max_steps", C.c_int32), ("youngs_ref", C.c_double), ("contact_nodes", ip),
                ("n_contact", C.c_int32), ("max_outer", C.c_int32), ("eps_phi", C.c_double),
                ("profile", C.c_int32), ("outer_warm", C.c_int32), ("contact_mode", C.c_int32),
                ("x0_predict", C.c_int32), ("lbfgs_warm", C.c_int32), ("plane_n", C.c_double * 3),
                ("plane_d", C.c_double)]


class PdStats(C.Structure):
    _fields_ = [("iters_fwd", ip), ("iters_adj", ip), ("contact_outer", ip), ("final_res_fwd", dp),
                ("final_res_adj", dp), ("n_nonconverged", C.c_int32)]


_lib = None


def load():
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2101_05917_b200.buildlib` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    lib.pd_create.argtypes = [C.POINTER(PdMesh), C.POINTER(PdMaterial), C.c_double, ip, C.c_int32,
                              C.POINTER(PdOptions), C.POINTER(vp)]
    lib.pd_forward.argtypes = [vp, C.c_int32, vp, vp, vp, C.c_int64, vp, vp, C.c_int32, vp, vp,
                               C.POINTER(PdStats), vp]
    lib.pd_backward.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, C.POINTER(PdStats), vp]
    lib.pd_backward_steps.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, C.POINTER(PdStats), vp]
    lib.pd_eval_objective.argtypes = [vp, C.c_int32, vp, vp, vp, vp, vp, vp, vp]
    lib.pd_apply_Ainv.argtypes = [vp, C.c_int32, vp, vp, vp]
    lib.pd_apply_AN.argtypes = [vp, C.c_int32, vp, vp, vp, vp, vp, vp]
    lib.pd_project_rotations.argtypes = [vp, C.c_int32, vp, vp, vp]
    lib.pd_polar_stats.argtypes = [vp, C.c_int32, vp, C.POINTER(C.c_int64), vp]
    lib.pd_info.argtypes = [vp, C.POINTER(C.c_int64), C.c_int32]
    lib.pd_profile.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32]
    lib.pd_contact_sets.argtypes = [vp, C.POINTER(C.c_uint8)]
    lib.pd_last_error.argtypes = [vp]
    lib.pd_last_error.restype = C.c_char_p
    lib.pd_destroy.argtypes = [vp]
    lib.pd_destroy.restype = None
    for name in EXPORTS:
        if name not in ("pd_last_error", "pd_destroy"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib
