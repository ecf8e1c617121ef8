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
