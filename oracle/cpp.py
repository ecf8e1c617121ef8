"""ctypes binding of libtilt_oracle.so (include/tilt_oracle.h): the C++17 fp64 oracle twin of
tilt_solve_batch. TEST INFRASTRUCTURE like the rest of oracle/: only tests/, __graft_entry__ and
bench.py's CPU baseline / reference arm use it. Built by __graft_entry__.build()."""
from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtilt_oracle.so")


class OracleParams(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("mu0_scale", ctypes.c_double), ("mu_max_ratio", ctypes.c_double),
                ("rho0", ctypes.c_double), ("eps1", ctypes.c_double), ("eps2", ctypes.c_double),
                ("obj_tol", ctypes.c_double), ("tau_tol", ctypes.c_double), ("max_inner", ctypes.c_int32),
                ("max_outer", ctypes.c_int32), ("constraints", ctypes.c_int32), ("vws", ctypes.c_int32),
                ("fixed_inner", ctypes.c_int32), ("fixed_outer", ctypes.c_int32)]


class OracleReport(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("stop_rule", ctypes.c_int32), ("outer_iters", ctypes.c_int32),
                ("inner_iters", ctypes.c_int32), ("rank", ctypes.c_int32), ("rank_band", ctypes.c_int32),
                ("jacobi_sweeps", ctypes.c_int32), ("objective", ctypes.c_double), ("crit1", ctypes.c_double),
                ("crit2", ctypes.c_double), ("patch_norm", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: python -c 'import __graft_entry__ as g; g.build()'")
        L = ctypes.CDLL(LIB_PATH)
        L.tilt_oracle_default_params.argtypes = [ctypes.POINTER(OracleParams)]
        L.tilt_oracle_solve_batch.restype = ctypes.c_int32
        L.tilt_oracle_solve_batch.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.POINTER(OracleParams), ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
        L.tilt_oracle_svt.restype = ctypes.c_int32
        L.tilt_oracle_svt.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                      ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def default_params(**kw) -> OracleParams:
    p = OracleParams()
    lib().tilt_oracle_default_params(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, "lambda_" if k == "lam" else k, v)
    return p


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def solve_batch(images, patch_image, boxes, tau0, kind, prm: OracleParams | None = None, n_threads: int = 0):
    """tilt_oracle_solve_batch on host arrays; returns (tau [B][p], A, E [B][m][n], reports (numpy struct))."""
    images = np.ascontiguousarray(images, dtype=np.float64)
    n_images, H, W = images.shape
    patch_image = np.ascontiguousarray(patch_image, dtype=np.int32)
    boxes = np.ascontiguousarray(boxes, dtype=np.int32)
    B = boxes.shape[0]
    p = 8 if kind == 1 else 6
    m, n = (int(boxes[0, 3]), int(boxes[0, 2])) if B else (0, 0)
    t0 = None if tau0 is None else np.ascontiguousarray(tau0, dtype=np.float64).reshape(B, p)
    tau = np.zeros((B, p))
    A = np.zeros((B, m, n))
    E = np.zeros((B, m, n))
    rep = (OracleReport * max(B, 1))()
    prm = prm if prm is not None else default_params()
    st = lib().tilt_oracle_solve_batch(_p(images), n_images, H, W, _p(patch_image), _p(boxes), _p(t0), B, kind,
                                       ctypes.byref(prm), _p(tau), _p(A), _p(E), ctypes.cast(rep, ctypes.c_void_p),
                                       n_threads)
    if st != 0:
        raise ValueError("tilt_oracle_solve_batch: invalid arguments")
    reps = np.ctypeslib.as_array(rep)[:B] if B else np.zeros(0)
    return tau, A, E, [{f: getattr(rep[b], f) for f, _ in OracleReport._fields_} for b in range(B)]


def svt(M, eps):
    """S_eps(M) by the C++ oracle's own Jacobi SVD: (A, sigma, sweeps)."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, n = M.shape
    A = np.zeros((m, n))
    sig = np.zeros(min(m, n))
    sw = lib().tilt_oracle_svt(_p(M), m, n, float(eps), _p(A), _p(sig))
    return A, sig, sw
