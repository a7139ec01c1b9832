"""ctypes declarations of include/helm.h (argument marshalling only).

Loading fails loudly if lib/libhelm.so is missing: there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libhelm.so")
# A/B tuning only: HELM_LIB_VARIANT=name loads lib/libhelm_<name>.so (an in-tree build of
# another revision of the same C ABI)
if os.environ.get("HELM_LIB_VARIANT"):
    LIB_PATH = os.path.join(_PKG, "lib", "libhelm_%s.so" % os.environ["HELM_LIB_VARIANT"])


class HelmGrid(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("n", C.c_int64 * 3), ("h", C.c_double), ("pml", (C.c_int32 * 2) * 3),
                ("stencil", C.c_int32)]


class HelmPml(C.Structure):
    _fields_ = [("R", C.c_double), ("power", C.c_int32), ("v_ref", C.c_double)]


class HelmMlOpts(C.Structure):
    _fields_ = [("levels", C.c_int32), ("ks_o", C.c_int32), ("ks_i", C.c_int32), ("kc_o", C.c_int32),
                ("kc_i", C.c_int32)]


class HelmSolveOpts(C.Structure):
    _fields_ = [("k_inner", C.c_int32), ("max_outer", C.c_int32), ("rtol", C.c_double), ("precond", C.c_int32)]


class HelmAcq(C.Structure):
    _fields_ = [("src_xyz", C.POINTER(C.c_double)), ("rec_xyz", C.POINTER(C.c_double)), ("kaiser_b", C.c_double),
                ("half_width", C.c_int32)]


class HelmSolveReport(C.Structure):
    _fields_ = [("outer_cycles", C.c_int32), ("converged", C.c_int32), ("rel_residual", C.c_double),
                ("matvecs", C.c_int64 * 4), ("bytes_alg", C.c_double)]

    def as_dict(self):
        return {"outer_cycles": self.outer_cycles, "converged": bool(self.converged),
                "rel_residual": self.rel_residual, "matvecs": list(self.matvecs), "bytes_alg": self.bytes_alg}


HELM_OK, HELM_ERR_ARG, HELM_ERR_SHAPE, HELM_ERR_CUDA, HELM_ERR_OOM, HELM_ERR_STATE = 0, -1, -2, -3, -4, -5
HELM_C64, HELM_C128 = 0, 1
HELM_STD2, HELM_OPT = 0, 1
NCLASS = 12
CLASS_NAMES = ["stencil", "stencil_resid", "norm", "arnoldi", "update", "solupdate", "copy", "restrict",
               "prolong_add", "fwi", "setup", "vcycle_persist"]

_P = C.c_void_p
_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_rep = C.POINTER(HelmSolveReport)

SIGNATURES = {
    "helm_setup": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_double, C.POINTER(HelmPml), C.c_int, C.c_int32,
                             C.POINTER(HelmMlOpts), _P, C.POINTER(_P)]),
    "helm_apply": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P]),
    "helm_solve": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, C.POINTER(HelmSolveOpts), _rep, _P]),
    "fwi_misfit_grad": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, C.c_int32,
                                  _i64, C.c_int32, _i64, _d, C.POINTER(HelmPml), C.c_int,
                                  C.POINTER(HelmSolveOpts), C.c_int32, _P, _rep, _P]),
    "fwi_forward": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, _i64,
                              C.c_int32, _i64, C.POINTER(HelmPml), C.c_int, C.POINTER(HelmSolveOpts),
                              C.c_int32, _d, _rep, _P]),
    "fwi_jacobian": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, _i64,
                               C.c_int32, _i64, _d, C.POINTER(HelmPml), C.c_int, C.POINTER(HelmSolveOpts),
                               C.c_int32, _d, _rep, _P]),
    "fwi_jacobian_adjoint": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32,
                                       C.c_int32, _i64, C.c_int32, _i64, _d, C.POINTER(HelmPml), C.c_int,
                                       C.POINTER(HelmSolveOpts), C.c_int32, _P, _rep, _P]),
    "fwi_gn_hessian": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, _i64,
                                 C.c_int32, _i64, _d, C.POINTER(HelmPml), C.c_int, C.POINTER(HelmSolveOpts),
                                 C.c_int32, _P, _rep, _P]),
    "fwi_misfit_grad_subset": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, C.c_int32,
                                         _i64, C.c_int32, _i64, _d, C.POINTER(C.c_uint8), C.POINTER(HelmPml), C.c_int,
                                         C.POINTER(HelmSolveOpts), C.c_int32, _P, _rep, _P]),
    "fwi_misfit_grad_acq": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.POINTER(HelmAcq), _d, C.POINTER(HelmPml), C.c_int,
                                      C.POINTER(HelmSolveOpts), C.c_int32, _P, _rep, _P]),
    "fwi_forward_acq": (C.c_int, [C.POINTER(HelmGrid), _d, C.c_int32, _d, _d, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.POINTER(HelmAcq), C.POINTER(HelmPml), C.c_int, C.POINTER(HelmSolveOpts),
                                  C.c_int32, _d, _rep, _P]),
    "helm_levels": (C.c_int, [_P, C.POINTER(C.c_int32), _i64]),
    "helm_get_level": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64, _d, _d]),
    "helm_vcycle": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P]),
    "helm_transfer": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P]),
    "helm_workspace_vectors": (C.c_double, [_P]),
    "helm_profile": (C.c_int, [C.c_int32, C.c_int32]),
    "helm_profile_read": (C.c_int, [C.c_int32, _i64, _i64, _d, _d]),
    "helm_probe_kernel": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _d, _P]),
    "helm_launch_count": (C.c_int64, []),
    "helm_destroy": (None, [_P]),
    "helm_last_error": (C.c_char_p, []),
    "helm_version": (C.c_char_p, []),
}

_lib = None


class HelmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"helm status {status}: {msg}")
        self.status = status


def load():
    """Load libhelm.so (building it first if nvcc is available and it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build
        build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libhelm.so not found at {LIB_PATH}; run `python -m paper_1703_09268_b200.build`")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != HELM_OK:
        raise HelmError(status, load().helm_last_error().decode())
