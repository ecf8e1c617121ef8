"""Evaluation of recovered transforms (used by tests and tools; not part of the method)."""
from __future__ import annotations

import numpy as np


def rectified(tau: np.ndarray, tau_g: np.ndarray, tol: float = 0.05) -> bool:
    """Success test of the range-of-convergence / corruption experiments (reading Z25): the
    recovered linear part L equals the planted A_G up to the symmetries that keep a rank-r
    axis-aligned texture axis-aligned — L = A_G P with P diagonal or anti-diagonal (axis scaling,
    axis swap) — to ``tol`` relative (off-pattern entries of A_G^{-1} L against its largest)."""
    lin = np.array([[tau[0], tau[1]], [tau[2], tau[3]]])
    ag = np.array([[tau_g[0], tau_g[1]], [tau_g[2], tau_g[3]]])
    p = np.linalg.solve(ag, lin)
    big = np.abs(p).max()
    if not np.isfinite(big) or big == 0:
        return False
    diag_off = max(abs(p[0, 1]), abs(p[1, 0])) / big
    anti_off = max(abs(p[0, 0]), abs(p[1, 1])) / big
    return bool(min(diag_off, anti_off) < tol)


def _h_of(tau: np.ndarray) -> np.ndarray:
    """3x3 matrix of a parameter vector (h11, h12, h21, h22, h13, h23[, h31, h32]) (reading Z16)."""
    h = np.eye(3)
    h[0, 0], h[0, 1], h[1, 0], h[1, 1], h[0, 2], h[1, 2] = tau[:6]
    if len(tau) == 8:
        h[2, 0], h[2, 1] = tau[6], tau[7]
    return h


def recovered_p9(tau: np.ndarray, tau_g: np.ndarray, off_tol: float = 0.02, persp_tol: float = 1e-2) -> bool:
    """tau* equals the planted H_G up to {translation, axis scaling}: the linear
    part of H_G^{-1} tau* is diagonal within ``off_tol`` relative and its perspective part is below
    ``persp_tol`` (the aspect direction is a null direction of TILT, reading Z10)."""
    h = np.linalg.solve(_h_of(np.asarray(tau_g, np.float64)), _h_of(np.asarray(tau, np.float64)))
    if not np.all(np.isfinite(h)) or h[2, 2] == 0:
        return False
    h = h / h[2, 2]
    lin = h[:2, :2]
    if lin[0, 0] == 0 or lin[1, 1] == 0:
        return False
    off = max(abs(lin[0, 1]) / abs(lin[0, 0]), abs(lin[1, 0]) / abs(lin[1, 1]))
    return bool(off < off_tol and max(abs(h[2, 0]), abs(h[2, 1])) < persp_tol)


def table2_error(tau: np.ndarray, tau_g: np.ndarray) -> float:
    """Table 2's error measure ||tau* - tau_G|| / ||tau_G||."""
    tau, tau_g = np.asarray(tau, np.float64), np.asarray(tau_g, np.float64)
    return float(np.linalg.norm(tau - tau_g) / np.linalg.norm(tau_g))


def agree_modulo_aspect(tau_a: np.ndarray, tau_b: np.ndarray, tol: float = 1e-3) -> bool:
    """tau_a equals tau_b up to TILT's null direction (reading Z10: low rank is invariant to axis
    scaling, and the area row leaves the aspect diag(s, 1/s) free): H_b^{-1} H_a, normalised, is
    diag(s, 1/s, 1) to ``tol`` (off-diagonal and perspective entries, and the area s (1/s) = 1)."""
    h = np.linalg.solve(_h_of(np.asarray(tau_b, np.float64)), _h_of(np.asarray(tau_a, np.float64)))
    if not np.all(np.isfinite(h)) or h[2, 2] == 0:
        return False
    h = h / h[2, 2]
    off = max(abs(h[0, 1]), abs(h[1, 0]), abs(h[0, 2]), abs(h[1, 2]), abs(h[2, 0]), abs(h[2, 1]))
    return bool(off < tol and abs(h[0, 0] * h[1, 1] - 1.0) < tol)
