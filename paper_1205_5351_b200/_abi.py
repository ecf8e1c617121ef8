"""ctypes mirror of include/tilt.h (argument marshalling only; every step runs in libtilt.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a). Importing this
module loads it and fails loudly if it is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TILT_LIB: alternative build of the same library (A/B experiments of kernel variants)
LIB_PATH = os.environ.get("TILT_LIB") or os.path.join(_HERE, "libtilt.so")

TILT_OK, TILT_E_ARG, TILT_E_CUDA, TILT_E_OOM, TILT_E_UNSUPPORTED = 0, 1, 2, 3, 4
AFFINE, HOMOGRAPHY = 0, 1
CONVERGED, MAX_OUTER, WINDOW_ESCAPE, SINGULAR_GRAM, ZERO_PATCH, DIVERGED, BAD_BOX = range(7)
CONSTRAINTS_NONE, CONSTRAINTS_CENTER_AREA = 0, 1


class TiltParams(ctypes.Structure):
    _fields_ = [
        ("lambda_", ctypes.c_float),
        ("mu0_scale", ctypes.c_float),
        ("mu_max_ratio", ctypes.c_float),
        ("rho0", ctypes.c_float),
        ("eps1", ctypes.c_float),
        ("eps2", ctypes.c_float),
        ("obj_tol", ctypes.c_float),
        ("tau_tol", ctypes.c_float),
        ("max_inner", ctypes.c_int32),
        ("max_outer", ctypes.c_int32),
        ("constraint_mode", ctypes.c_int32),
        ("vws", ctypes.c_int32),
        ("svd_warm", ctypes.c_int32),
        ("pyramid_levels", ctypes.c_int32),
        ("jacobi_tol", ctypes.c_float),
        ("jacobi_max_sweeps", ctypes.c_int32),
        ("fixed_inner_iters", ctypes.c_int32),
        ("fixed_outer_iters", ctypes.c_int32),
        ("rho_replay", ctypes.c_void_p),
        ("trace", ctypes.c_void_p),
        ("win_h", ctypes.c_int32),
        ("win_w", ctypes.c_int32),
        ("kernel_path", ctypes.c_int32),
        ("ns_period", ctypes.c_int32),
        ("inner_solver", ctypes.c_int32),
        ("adm_rho", ctypes.c_float),
        ("adm_tol", ctypes.c_float),
        ("ctas_per_sm", ctypes.c_int32),
        ("pyramid_warm", ctypes.c_int32),
        ("svd_mode", ctypes.c_int32),
        ("svd_ws_gate", ctypes.c_float),
    ]


class TiltReport(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("stop_rule", ctypes.c_int32),
        ("outer_iters", ctypes.c_int32),
        ("inner_iters", ctypes.c_int32),
        ("jacobi_sweeps", ctypes.c_int32),
        ("aux_sweeps", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("rank_band", ctypes.c_int32),
        ("svt_rank", ctypes.c_int32),
        ("sweep_cap_hits", ctypes.c_int32),
        ("objective", ctypes.c_float),
        ("crit1", ctypes.c_float),
        ("crit2", ctypes.c_float),
        ("patch_norm", ctypes.c_float),
        ("dtau_inf", ctypes.c_float),
        ("mu_last", ctypes.c_float),
        ("jacobi_rotations", ctypes.c_int32),
        ("kernel_path", ctypes.c_int32),
        ("svd_warm_steps", ctypes.c_int32),
    ]


REPORT_FIELDS = [f[0] for f in TiltReport._fields_]
REPORT_BYTES = ctypes.sizeof(TiltReport)


class TiltCreateOpts(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("max_batch", ctypes.c_int32),
        ("max_m", ctypes.c_int32),
        ("max_n", ctypes.c_int32),
        ("max_p", ctypes.c_int32),
        ("max_image_elems", ctypes.c_int64),
    ]


EXPORTS = [
    "tilt_abi_version", "tilt_status_string", "tilt_patch_status_string", "tilt_last_error",
    "tilt_default_params", "tilt_create", "tilt_destroy", "tilt_set_stream", "tilt_solve_batch",
    "tilt_solve_batch_host", "tilt_warp_batch", "tilt_svt_batch", "tilt_project_batch",
    "tilt_inner_batch", "tilt_launch_count", "tilt_set_svt_path",
]

_P = ctypes.c_void_p
_I = ctypes.c_int32


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.tilt_abi_version.restype = _I
    lib.tilt_status_string.restype = ctypes.c_char_p
    lib.tilt_status_string.argtypes = [_I]
    lib.tilt_patch_status_string.restype = ctypes.c_char_p
    lib.tilt_patch_status_string.argtypes = [_I]
    lib.tilt_last_error.restype = ctypes.c_char_p
    lib.tilt_default_params.restype = _I
    lib.tilt_default_params.argtypes = [ctypes.POINTER(TiltParams)]
    lib.tilt_create.restype = _I
    lib.tilt_create.argtypes = [ctypes.POINTER(_P), ctypes.POINTER(TiltCreateOpts)]
    lib.tilt_destroy.restype = _I
    lib.tilt_destroy.argtypes = [_P]
    lib.tilt_set_stream.restype = _I
    lib.tilt_set_stream.argtypes = [_P, _P]
    lib.tilt_solve_batch.restype = _I
    lib.tilt_solve_batch.argtypes = [_P, _P, _I, _I, _I, _P, _P, _P, _I, _I, ctypes.POINTER(TiltParams),
                                     _P, _P, _P, _P, _P]
    lib.tilt_solve_batch_host.restype = _I
    lib.tilt_solve_batch_host.argtypes = [_P, _P, _I, _I, _I, _P, _P, _P, _I, _I,
                                          ctypes.POINTER(TiltParams), _P, _P, _P, _P]
    lib.tilt_warp_batch.restype = _I
    lib.tilt_warp_batch.argtypes = [_P, _P, _I, _I, _I, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]
    lib.tilt_svt_batch.restype = _I
    lib.tilt_svt_batch.argtypes = [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P]
    lib.tilt_project_batch.restype = _I
    lib.tilt_project_batch.argtypes = [_P, _P, _P, _I, _P, _I, _I, _I, _I, _P, _P, _P]
    lib.tilt_inner_batch.restype = _I
    lib.tilt_inner_batch.argtypes = [_P, _P, _P, _P, _I, _I, _I, _I, _I, ctypes.POINTER(TiltParams),
                                     _P, _P, _P, _P]
    lib.tilt_launch_count.restype = ctypes.c_int64
    lib.tilt_launch_count.argtypes = [_P]
    lib.tilt_set_svt_path.restype = _I
    lib.tilt_set_svt_path.argtypes = [_P, _I]
    return lib


lib = _load()


class TiltError(RuntimeError):
    pass


def check(status: int, what: str = "") -> None:
    if status != TILT_OK:
        msg = lib.tilt_status_string(status).decode()
        detail = lib.tilt_last_error().decode()
        raise TiltError(f"{what}: {msg} {detail}".strip())


def default_params(**overrides) -> TiltParams:
    prm = TiltParams()
    check(lib.tilt_default_params(ctypes.byref(prm)), "tilt_default_params")
    for k, v in overrides.items():
        key = "lambda_" if k in ("lambda", "lam") else k
        if not hasattr(prm, key):
            raise KeyError(k)
        setattr(prm, key, v)
    return prm
