"""Plain fp64 CPU oracle for the TILT hot path of Ren & Lin, arXiv 1205.5351.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import or run this module. The product path
(``paper_1205_5351_b200``) never imports it, and this module imports nothing from the product.

Every function follows the paper step by step in its notation; citations are ``P:<line>`` of
``/root/reference/PAPER.md`` with the section / equation label. Where the paper is silent or
garbled the reading taken is named (R*/Z*/E*), listed in DESIGN.md "Readings of the paper".
Library primitives used as single steps: ``numpy.linalg.svd`` (the SVD in Eq. S_operator; the
oracle's own one-sided Jacobi ``jacobi_svd`` is the alternative, Params.svd = "jacobi"),
``numpy.linalg.cholesky`` / ``solve`` (the p x p Gram system of Eq. Jperpv). No blocking, fusion or
reordering beyond what the equations state.

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` (see DESIGN.md table
"Oracle pins"); nothing is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

AFFINE = 0
HOMOGRAPHY = 1

# per-patch status codes (mirrors include/tilt.h tilt_patch_status; values are the ABI's)
CONVERGED = 0
MAX_OUTER = 1
WINDOW_ESCAPE = 2
SINGULAR_GRAM = 3
ZERO_PATCH = 4
DIVERGED = 5

# outer stop rules (reading Z9)
STOP_NONE, STOP_OBJECTIVE, STOP_DTAU, STOP_MAX_OUTER = 0, 1, 2, 3


@dataclass
class Params:
    """Defaults of DESIGN.md "Readings"; the paper states none of them."""

    lam: float = -1.0           # <= 0 -> 1/sqrt(max(m, n))  (reading Z8)
    mu0_scale: float = 1.25     # mu0 = mu0_scale / sigma_1(D_hat)  (Z3)
    mu_max_ratio: float = 1e6   # mu_max = ratio * mu0  (Z6)
    rho0: float = 2.0           # Eq. rho, P:454-463  (Z7)
    eps1: float = 1e-6          # Eq. Cond1, P:489-492 (Z7)
    eps2: float = 0.1           # Eq. Cond2 / Eq. rho (Z7)
    obj_tol: float = 1e-5       # outer stop, relative objective change (Z9)
    tau_tol: float = 1e-4       # outer stop, ||dtau||_inf (Z9)
    max_inner: int = 1000
    max_outer: int = 50
    constraints: bool = True    # Q = centre + area rows (Z10)
    vws: bool = True            # variable warm start (Eq. warm_start)
    fixed_inner_iters: int = 0  # >0: run exactly K inner iterations (test mode)
    fixed_outer_iters: int = 0  # >0: run exactly F outer iterations (test mode)
    svd: str = "lapack"         # SVD inside S_eps: "lapack" (library step) or "jacobi" (own, jacobi_svd)
    inner: str = "ladmap"       # inner solver: "ladmap" (the paper's) or "adm" (the baseline of P:241-264)
    adm_rho: float = 1.25       # ADM penalty growth mu_{k+1} = rho mu_k, unbounded (reading Z24)
    adm_tol: float = 1e-6       # ADM stop: ||D + J dtau - A - E||_F / ||D||_F < adm_tol (reading Z24;
                                # 1e-7 reproduces Table 1's ADM counts in fp64, 1e-6 is fp32-resolvable)
    pyramid_warm: bool = False  # 2-level pyramid: the fine level's first inner loop starts from the
                                # coarse A, E, Y upsampled (reading Z26)
    tau_noise: float = 0.0      # test instrumentation (reading Z22): tau <- tau (1 + tau_noise N(0,1))
                                # after every outer update, seeded by noise_seed -- the chain
                                # sensitivity of the outer loop to per-step differences; 0 = exact
    crit_noise: float = 0.0     # test instrumentation (reading Z22): Cond1's statistic is compared as
    noise_seed: int = 0         # crit1 (1 + crit_noise N(0,1)) -- the relative resolution of an fp32
                                # crit1 near eps1 -- to classify decision-sensitive patches; 0 = exact


# ----------------------------------------------------------------------------------------------
# Proximal operators
# ----------------------------------------------------------------------------------------------

def shrink(x, eps):
    """Scalar shrinkage T_eps(x) = sgn(x) max(|x| - eps, 0)  (P:482, P:484-488 Eq. E_1)."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.maximum(np.abs(x) - eps, 0.0)


def jacobi_svd(w, tol=1e-14, max_sweeps=60, v0=None):
    """The oracle's own SVD: one-sided (Hestenes) Jacobi in fp64 (SURVEY.md §8(c) oracle step 5).

    B = W V with V orthogonal (identity, or the warm start v0); every sweep visits each column pair
    (i, j) once (round-robin parallel ordering: the n/2 disjoint pairs of a round are rotated
    together), rotating the pair so that b_i . b_j = 0 with the smaller-angle tangent
    t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = (beta - alpha)/(2 gamma); a pair is skipped
    when |gamma| <= tol sqrt(alpha beta). Stops after a sweep without rotation (<= max_sweeps).
    Returns (U, sigma, V, sweeps): W = U diag(sigma) V^T, sigma descending; columns of U for
    sigma = 0 are 0 (they multiply zero in every use below).
    """
    b = np.array(w, dtype=np.float64, copy=True)
    m, n = b.shape
    v = np.eye(n) if v0 is None else np.array(v0, dtype=np.float64, copy=True)
    if v0 is not None:
        b = b @ v
    nn = n + (n & 1)
    q = nn - 1
    # columns below this squared norm are zero to working precision (the n - rank columns of a
    # rank-deficient W converge to rounding noise, which must not keep the sweeps going)
    small = (n * np.finfo(np.float64).eps * max(np.linalg.norm(b), np.finfo(np.float64).tiny)) ** 2
    sweeps = 0
    for sweeps in range(1, max_sweeps + 1):
        rotated = False
        for r in range(q):
            k = np.arange(nn // 2)
            i = np.where(k == 0, q, (r + k) % q)
            j = np.where(k == 0, r % q, (r - k) % q)
            keep = (i < n) & (j < n)
            i, j = i[keep], j[keep]
            bi, bj = b[:, i], b[:, j]
            alpha = np.einsum("ij,ij->j", bi, bi)
            beta = np.einsum("ij,ij->j", bj, bj)
            gamma = np.einsum("ij,ij->j", bi, bj)
            act = (np.abs(gamma) > tol * np.sqrt(alpha * beta)) & (alpha > small) & (beta > small)
            if not np.any(act):
                continue
            rotated = True
            i, j, alpha, beta, gamma = i[act], j[act], alpha[act], beta[act], gamma[act]
            zeta = (beta - alpha) / (2.0 * gamma)
            t = np.sign(zeta) / (np.abs(zeta) + np.hypot(1.0, zeta))
            t[zeta == 0.0] = 1.0
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = c * t
            bi, bj = b[:, i].copy(), b[:, j].copy()
            b[:, i] = c * bi - s * bj
            b[:, j] = s * bi + c * bj
            vi, vj = v[:, i].copy(), v[:, j].copy()
            v[:, i] = c * vi - s * vj
            v[:, j] = s * vi + c * vj
        if not rotated:
            break
    sigma = np.sqrt(np.einsum("ij,ij->j", b, b))
    order = np.argsort(-sigma, kind="stable")
    sigma, b, v = sigma[order], b[:, order], v[:, order]
    u = np.divide(b, sigma, out=np.zeros_like(b), where=sigma > 0)
    return u, sigma, v, sweeps


SVD_METHOD = {"lapack": None, "jacobi": jacobi_svd}


def svt(w, eps, method="lapack"):
    """Singular value shrinkage S_eps(W) = U T_eps(Sigma) V^T  (Eqs. A_1, S_operator).

    The SVD is the library routine (method="lapack", a single library step) or the oracle's own
    one-sided Jacobi (method="jacobi", ``jacobi_svd``); both give the same S_eps(W) (the prox of
    eps ||.||_*, is single valued). Returns (S_eps(W), sigma(W)) with sigma descending.
    """
    w = np.asarray(w, dtype=np.float64)
    if method == "jacobi":
        u, sig, v, _ = jacobi_svd(w)
        return (u * shrink(sig, eps)) @ v.T, sig
    try:
        u, sig, vt = np.linalg.svd(w, full_matrices=False)
    except np.linalg.LinAlgError:  # LAPACK's divide and conquer did not converge: the oracle's own SVD
        u, sig, v, _ = jacobi_svd(w)
        return (u * shrink(sig, eps)) @ v.T, sig
    return (u * shrink(sig, eps)) @ vt, sig


def nuclear_norm(a):
    """||A||_* = sum of singular values."""
    return float(np.linalg.svd(np.asarray(a, dtype=np.float64), compute_uv=False).sum())


def objective(a, e, lam):
    """||A||_* + lambda ||E||_1  (Eq. TILT_2)."""
    return nuclear_norm(a) + lam * float(np.abs(e).sum())


# ----------------------------------------------------------------------------------------------
# D o tau and its Jacobian (Alg. 1 Step 1; readings R1-R4 = Z2, Z15, Z16)
# ----------------------------------------------------------------------------------------------

def frame(box):
    """Normalised frame of the window (reading Z15): centre c, scale s, pixel offsets du, dv."""
    x0, y0, w, h = (int(v) for v in box)
    m, n = h, w
    s = max(m, n) / 2.0
    cx = x0 + (n - 1) / 2.0
    cy = y0 + (m - 1) / 2.0
    dv = (np.arange(m, dtype=np.float64) - (m - 1) / 2.0)[:, None] * np.ones((1, n))
    du = (np.arange(n, dtype=np.float64) - (n - 1) / 2.0)[None, :] * np.ones((m, 1))
    return m, n, s, cx, cy, du, dv


def tau_to_h(tau, kind):
    """(h11, h12, h21, h22, h13, h23[, h31, h32]) -> 3x3 matrix (reading Z16)."""
    t = np.asarray(tau, dtype=np.float64)
    h31, h32 = (t[6], t[7]) if kind == HOMOGRAPHY else (0.0, 0.0)
    return np.array([[t[0], t[1], t[4]], [t[2], t[3], t[5]], [h31, h32, 1.0]])


def warp(image, box, tau, kind):
    """D o tau (bilinear) and J_raw = d(D o tau)/d tau.

    Source point of window pixel (i, j): x = (h11 u + h12 v + h13)/w, y = (h21 u + h22 v + h23)/w,
    w = h31 u + h32 v + 1 in the normalised frame (Z15, Z16). The Jacobian is the exact derivative
    of the bilinear interpolant taken from the same 4 taps (Z2), chained through the transform.
    Returns (d [m, n], J_raw [p, m, n], status); status WINDOW_ESCAPE if any 4-tap stencil leaves
    the image.
    """
    img = np.asarray(image, dtype=np.float64)
    hh, ww = img.shape
    m, n, s, cx, cy, du, dv = frame(box)
    h = tau_to_h(tau, kind)
    p = 6 if kind == AFFINE else 8
    w = 1.0 + (h[2, 0] * du + h[2, 1] * dv) / s
    xs = cx + (h[0, 0] * du + h[0, 1] * dv + s * h[0, 2]) / w
    ys = cy + (h[1, 0] * du + h[1, 1] * dv + s * h[1, 2]) / w
    if not (np.all(np.isfinite(xs)) and np.all(np.isfinite(ys))):
        return None, None, WINDOW_ESCAPE
    x0 = np.floor(xs)
    y0 = np.floor(ys)
    if x0.min() < 0 or x0.max() + 1 > ww - 1 or y0.min() < 0 or y0.max() + 1 > hh - 1:
        return None, None, WINDOW_ESCAPE
    fx = xs - x0
    fy = ys - y0
    xi = x0.astype(np.int64)
    yi = y0.astype(np.int64)
    i00 = img[yi, xi]
    i01 = img[yi, xi + 1]
    i10 = img[yi + 1, xi]
    i11 = img[yi + 1, xi + 1]
    d = (1 - fy) * ((1 - fx) * i00 + fx * i01) + fy * ((1 - fx) * i10 + fx * i11)
    # exact derivative of the bilinear interpolant w.r.t. pixel coordinates (Z2)
    dX = (1 - fy) * (i01 - i00) + fy * (i11 - i10)
    dY = (1 - fx) * (i10 - i00) + fx * (i11 - i01)
    # chain rule to the normalised frame: x = (X - cx)/s  =>  dI/dx = s dI/dX
    u = du / s
    v = dv / s
    xn = (xs - cx) / s
    yn = (ys - cy) / s
    ix = s * dX
    iy = s * dY
    # dx/dh11 = u/w, dx/dh12 = v/w, dx/dh13 = 1/w, dx/dh31 = -x u/w, dx/dh32 = -x v/w (same for y)
    cols = [ix * u / w, ix * v / w, iy * u / w, iy * v / w, ix / w, iy / w]
    if kind == HOMOGRAPHY:
        cols += [-(ix * xn + iy * yn) * u / w, -(ix * xn + iy * yn) * v / w]
    jraw = np.stack(cols)
    assert jraw.shape[0] == p
    return d, jraw, CONVERGED


def normalise(d, jraw):
    """Alg. 1 Step 1: D_hat = d/||d||_F, J = d/dzeta (D o zeta/||D o zeta||_F).

    Quotient rule: J = (J_raw - D_hat (D_hat^T J_raw)) / ||d||_F.
    """
    nd = float(np.linalg.norm(d))
    dh = d / nd
    c = np.tensordot(jraw, dh, axes=([1, 2], [0, 1]))  # D_hat^T J_raw, one entry per parameter
    j = (jraw - c[:, None, None] * dh[None, :, :]) / nd
    return dh, j, nd


def constraints_q(tau, kind, m, n):
    """Q (l=3 rows): centre x, centre y and area of the transformed window (Z10).

    Centre = tau(0, 0) = (h13, h23): rows are the unit vectors on h13, h23. Area = shoelace area of
    tau applied to the window corners (+-n/N, +-m/N), N = max(m, n); its gradient w.r.t. tau is
    taken analytically (quotient rule per corner). Each row is scaled to unit norm.
    """
    p = 6 if kind == AFFINE else 8
    h = tau_to_h(tau, kind)
    big = max(m, n)
    cu, cv = n / big, m / big
    corners = [(-cu, -cv), (cu, -cv), (cu, cv), (-cu, cv)]
    pts, grads = [], []
    for (u, v) in corners:
        w = h[2, 0] * u + h[2, 1] * v + 1.0
        x = (h[0, 0] * u + h[0, 1] * v + h[0, 2]) / w
        y = (h[1, 0] * u + h[1, 1] * v + h[1, 2]) / w
        gx = np.zeros(p)
        gy = np.zeros(p)
        gx[0], gx[1], gx[4] = u / w, v / w, 1.0 / w
        gy[2], gy[3], gy[5] = u / w, v / w, 1.0 / w
        if kind == HOMOGRAPHY:
            gx[6], gx[7] = -x * u / w, -x * v / w
            gy[6], gy[7] = -y * u / w, -y * v / w
        pts.append((x, y))
        grads.append((gx, gy))
    garea = np.zeros(p)
    for k in range(4):
        (xa, ya), (xb, yb) = pts[k], pts[(k + 1) % 4]
        (gxa, gya), (gxb, gyb) = grads[k], grads[(k + 1) % 4]
        # area = 1/2 sum_k (x_k y_{k+1} - x_{k+1} y_k)
        garea += 0.5 * (gxa * yb + xa * gyb - gxb * ya - xb * gya)
    q = np.zeros((3, p))
    q[0, 4] = 1.0
    q[1, 5] = 1.0
    q[2] = garea / np.linalg.norm(garea)
    return q


def shoelace_area(tau, kind, m, n):
    """Area of tau(window corners), the quantity whose gradient is Q's third row (test helper)."""
    h = tau_to_h(tau, kind)
    big = max(m, n)
    cu, cv = n / big, m / big
    pts = []
    for (u, v) in [(-cu, -cv), (cu, -cv), (cu, cv), (-cu, cv)]:
        w = h[2, 0] * u + h[2, 1] * v + 1.0
        pts.append(((h[0, 0] * u + h[0, 1] * v + h[0, 2]) / w, (h[1, 0] * u + h[1, 1] * v + h[1, 2]) / w))
    return 0.5 * sum(pts[k][0] * pts[(k + 1) % 4][1] - pts[(k + 1) % 4][0] * pts[k][1] for k in range(4))


# ----------------------------------------------------------------------------------------------
# The operator W^T W = I - J (J^T J + Q^T Q)^{-1} J^T  (P:587-606 Eq. Jperpv)
# ----------------------------------------------------------------------------------------------

class Projector:
    """W^T W applied implicitly: v - J((J^T J + Q^T Q)^{-1}(J^T v))  (Eq. Jperpv, Eq. WTW_property).

    With Q = None this is J_perp = I - J (J^T J)^{-1} J^T. ``count`` instruments the number
    of applications (two per LADMAP iteration).
    """

    class SingularGram(Exception):
        pass

    def __init__(self, j, q=None):
        j = np.asarray(j, dtype=np.float64)
        self.shape = j.shape[1:]
        self.jm = j.reshape(j.shape[0], -1).T  # mn x p ("arranged in an mn x p matrix")
        g = self.jm.T @ self.jm
        if q is not None:
            q = np.asarray(q, dtype=np.float64)
            g = g + q.T @ q
        self.q = q
        self.g = g
        try:
            self.chol = np.linalg.cholesky(g)  # "(J^T J)^{-1} ... can be pre-computed"
        except np.linalg.LinAlgError as exc:
            raise Projector.SingularGram(str(exc)) from exc
        if not np.all(np.isfinite(self.chol)) or np.min(np.diag(self.chol)) <= 0:
            raise Projector.SingularGram("non-positive pivot")
        self.count = 0

    def _gsolve(self, r):
        y = np.linalg.solve(self.chol, r)
        return np.linalg.solve(self.chol.T, y)

    def apply(self, v):
        """W^T W v for an m x n matrix v (vectorised row-major, reading Z1)."""
        self.count += 1
        vv = np.asarray(v, dtype=np.float64).reshape(-1)
        out = vv - self.jm @ self._gsolve(self.jm.T @ vv)
        return out.reshape(self.shape)

    def delta_tau(self, r):
        """Delta tau* = (J^T J + Q^T Q)^{-1} J^T r  (Eq. Delta_tau P:376-378 with Q)."""
        return self._gsolve(self.jm.T @ np.asarray(r, dtype=np.float64).reshape(-1))


# ----------------------------------------------------------------------------------------------
# SVD with warm start (Algorithm 2; Appendix A)
# ----------------------------------------------------------------------------------------------

def svd_warm_start(m_k, u, sig, v):
    """One Taylor step of Algorithm 2 along the Cayley curve of Eq. curve_to_search.

    (u, sig, v): the (approximate) SVD of M_{k-1}, u m x n column-orthonormal, sig the diagonal
    of Sigma (entries may be negative), v n x n orthogonal; m >= n. Steps:
      W = U Sigma V^T;  P_U = W M^T - M W^T,  P_V = W^T M - M^T W,  P_Sigma = diag(Sigma - U^T M V)
        (Eqs. projected_gradient1-3)
      h(0) = M - W,  h'(0) = P_U W + U P_Sigma V^T - W P_V,  Z = h'(0) + U P_Sigma V^T,
      h''(0) = -P_U Z + Z P_V
      f'(0) = <h(0), h'(0)>,  f''(0) = ||h'(0)||^2 + <h(0), h''(0)>,  t* = -f'(0)/f''(0)  (Eq. ft)
      U(t*) = (I + t*/2 P_U)^{-1}(I - t*/2 P_U) U,  Sigma(t*) = Sigma - t* P_Sigma,
      V(t*) = (I + t*/2 P_V)^{-1}(I - t*/2 P_V) V  (Eq. curve_to_search)
    Returns (U(t*), Sigma(t*), V(t*), t*); t* = 0 when f''(0) <= 0 (no descent model).
    """
    m_k = np.asarray(m_k, dtype=np.float64)
    w = (u * sig) @ v.T
    p_u = w @ m_k.T - m_k @ w.T
    p_v = w.T @ m_k - m_k.T @ w
    p_s = sig - np.einsum("ij,ij->j", u, m_k @ v)
    h0 = m_k - w
    ups = (u * p_s) @ v.T
    h1 = p_u @ w + ups - w @ p_v
    z = h1 + ups
    h2 = -p_u @ z + z @ p_v
    f1 = float(np.sum(h0 * h1))
    f2 = float(np.sum(h1 * h1) + np.sum(h0 * h2))
    t = -f1 / f2 if f2 > 0.0 else 0.0
    im, in_ = np.eye(p_u.shape[0]), np.eye(p_v.shape[0])
    u_t = np.linalg.solve(im + 0.5 * t * p_u, (im - 0.5 * t * p_u) @ u)
    v_t = np.linalg.solve(in_ + 0.5 * t * p_v, (in_ - 0.5 * t * p_v) @ v)
    return u_t, sig - t * p_s, v_t, t


def cayley_objective(m_k, u, sig, v, t):
    """f(t) = 1/2 ||M - U(t) Sigma(t) V(t)^T||_F^2 on the curve of Eq. curve_to_search (Eq. solve_t);
    test helper for the derivative formulas of Appendix A."""
    w = (u * sig) @ v.T
    p_u = w @ m_k.T - m_k @ w.T
    p_v = w.T @ m_k - m_k.T @ w
    p_s = sig - np.einsum("ij,ij->j", u, m_k @ v)
    im, in_ = np.eye(p_u.shape[0]), np.eye(p_v.shape[0])
    u_t = np.linalg.solve(im + 0.5 * t * p_u, (im - 0.5 * t * p_u) @ u)
    v_t = np.linalg.solve(in_ + 0.5 * t * p_v, (in_ - 0.5 * t * p_v) @ v)
    r = m_k - (u_t * (sig - t * p_s)) @ v_t.T
    return 0.5 * float(np.sum(r * r))


class SvdWarm:
    """The SVD warm start of LADMAP+SVDWS (Algorithm 2): keeps the previous (approximate) SVD and
    M_{k-1}; S_eps(M_k) uses one ``svd_warm_start`` step when ||M_k - M_{k-1}||_F < eps_svd, else a
    full SVD ("Else do full svd"). m < n is handled on the transpose (S_eps(M^T) = S_eps(M)^T).
    Reading Z27: a gated step is rejected (full SVD instead) only when f''(0) <= 0. Eq. ft
     replaces f by its quadratic model f(0) + f'(0) t + f''(0) t^2 / 2, whose stationary
    point t~* = -f'(0)/f''(0) is its minimiser only when f''(0) > 0 (for f''(0) <= 0 the model has no
    minimiser and the paper's bound ||U(t~*)Sigma(t~*)V(t~*)^T - M_k|| <= ||M_{k-1} - M_k||, P:921-935,
    has nothing to stand on). Any other t* is taken as printed: (I + t/2 P) is invertible for every
    skew P and the Cayley curve is feasible for every t, so no step-size rule applies.
    ``decisions`` logs 1 (warm step) / 0 (full SVD) per call."""

    def __init__(self, eps_svd):
        self.eps_svd = eps_svd
        self.prev = None
        self.m_prev = None
        self.warm_steps = 0
        self.full_svds = 0
        self.decisions = []
        self.cayley_sizes = []  # test instrumentation: max ||(t*/2) P_U||_F, ||(t*/2) P_V||_F per warm step

    def svt(self, m_k, eps):
        m_k = np.asarray(m_k, dtype=np.float64)
        tr = m_k.shape[0] < m_k.shape[1]
        x = m_k.T if tr else m_k
        step = None
        if self.prev is not None and np.linalg.norm(x - self.m_prev) < self.eps_svd:
            u, sig, v, t = svd_warm_start(x, *self.prev)
            if t != 0.0:
                step = (u, sig, v)
                w = (self.prev[0] * self.prev[1]) @ self.prev[2].T
                self.cayley_sizes.append(0.5 * abs(t) * max(np.linalg.norm(w @ x.T - x @ w.T),
                                                            np.linalg.norm(w.T @ x - x.T @ w)))
        if step is not None:
            u, sig, v = step
            self.warm_steps += 1
            self.decisions.append(1)
        else:
            u, sig, vt = np.linalg.svd(x, full_matrices=False)
            v = vt.T
            self.full_svds += 1
            self.decisions.append(0)
        self.prev = (u, sig, v)
        self.m_prev = x.copy()
        a = (u * shrink(sig, eps)) @ v.T
        return (a.T if tr else a), np.sort(np.abs(sig))[::-1]


# ----------------------------------------------------------------------------------------------
# LADMAP inner loop (P:437-468 Eqs. A, E, Y, mu, rho; P:489-497 Cond1/2; P:708-749 Eq. newvars2)
# ----------------------------------------------------------------------------------------------

@dataclass
class InnerResult:
    A: np.ndarray
    E: np.ndarray
    Y: np.ndarray
    iters: int
    mu: float               # mu_k used by the last iteration's updates
    sigma_m: np.ndarray     # singular values of the last M_k (so sigma(A) = T_{1/mu}(sigma_m))
    crit1: float
    crit2: float
    trace: list = field(default_factory=list)   # (mu_k, crit1, crit2, rho_bit) per iteration
    converged: bool = False


def ladmap(dh, proj, lam, mu0, mu_max, rho0, eps1, eps2, max_inner, a0, e0, y0,
           fixed_iters=0, rho_replay=None, svd="lapack", crit_noise=None):
    """LADMAP for min ||A||_* + lam ||E||_1  s.t.  W^T W (A + E) = W^T W D  (Eq. reformulated_TILT2).

    Iteration (Eq. newvars2, with errata E1 (+ sign of the dual step, as Eq. Y)
    and E2 (N_k starts from E_k, as P:451 / Eq. update_y' P:343-347)):
        M_k     = A_k - Y_k/mu_k - W^TW(A_k + E_k - D)
        A_{k+1} = S_{1/mu_k}(M_k)                                   (Eq. A_1)
        N_k     = E_k - Y_k/mu_k - W^TW(A_{k+1} + E_k - D)
        E_{k+1} = T_{lam/mu_k}(N_k)                                 (Eq. E_1)
        Y_{k+1} = Y_k + mu_k W^TW(A_{k+1} + E_{k+1} - D)            (Eq. newvars2 / Eq. Y)
        rho     = rho0 if mu_k max(||dA||, ||dE||)/||W^TW D|| < eps2 else 1   (Eq. rho)
        mu_{k+1} = min(mu_max, rho mu_k)                             (Eq. mu)
    The product W^TW(A_{k+1}+E_{k+1}-D) is reused for the next M, so two
    projector applications are made per iteration. Stop when Cond1 and Cond2 hold (P:489-497,
    strict inequalities, reading Z12), unless ``fixed_iters`` > 0 (test mode).
    ``rho_replay`` (sequence of 0/1) overrides the rho decision (parity protocol, reading Z21).
    ``crit_noise`` = (scale, numpy Generator) perturbs the statistic Cond1 tests (test
    instrumentation of reading Z22: the stop decision as resolved by fp32 arithmetic); None = exact.
    """
    denom = float(np.linalg.norm(proj.apply(dh)))
    if denom == 0.0:  # D in span(J): the crit denominators degenerate; use 1 (reading R9)
        denom = 1.0
    a, e, y = a0.copy(), e0.copy(), y0.copy()
    r = proj.apply(a + e - dh)
    mu = mu0
    trace = []
    n_iter = fixed_iters if fixed_iters > 0 else max_inner
    crit1 = crit2 = float("nan")
    sig = None
    converged = False
    k = 0
    for k in range(n_iter):
        m_k = a - y / mu - r
        a1, sig = svd.svt(m_k, 1.0 / mu) if isinstance(svd, SvdWarm) else svt(m_k, 1.0 / mu, svd)
        n_k = e - y / mu - proj.apply(a1 + e - dh)
        e1 = shrink(n_k, lam / mu)
        r = proj.apply(a1 + e1 - dh)
        y = y + mu * r
        crit1 = float(np.linalg.norm(r)) / denom
        crit2 = mu * max(float(np.linalg.norm(a1 - a)), float(np.linalg.norm(e1 - e))) / denom
        a, e = a1, e1
        c1_test = crit1 if crit_noise is None else crit1 * (1.0 + crit_noise[0] * crit_noise[1].standard_normal())
        rho_bit = 1 if crit2 < eps2 else 0
        if rho_replay is not None and k < len(rho_replay):
            rho_bit = int(rho_replay[k])
        trace.append((mu, crit1, crit2, rho_bit))
        mu_used = mu
        if c1_test < eps1 and crit2 < eps2:
            converged = True
            if fixed_iters <= 0:
                return InnerResult(a, e, y, k + 1, mu_used, sig, crit1, crit2, trace, True)
        mu = min(mu_max, (rho0 if rho_bit else 1.0) * mu)
    return InnerResult(a, e, y, n_iter, trace[-1][0] if trace else mu, sig, crit1, crit2, trace,
                       converged)


# ----------------------------------------------------------------------------------------------
# ADM baseline inner loop (Zhang et al., as restated in P:241-264)
# ----------------------------------------------------------------------------------------------

@dataclass
class AdmResult:
    A: np.ndarray
    E: np.ndarray
    Y: np.ndarray
    dtau: np.ndarray
    iters: int
    mu: float               # mu_k of the last iteration's updates
    sigma_m: np.ndarray     # singular values of the last SVT argument
    resid: float            # ||D + J dtau - A - E||_F / ||D||_F at exit
    converged: bool = False


def adm(dh, proj, lam, mu0, rho, tol, max_inner, fixed_iters=0):
    """Gauss-Seidel ADM on the augmented Lagrangian of Eq. TILT_3:
        A_{k+1}   = argmin_A L = S_{1/mu_k}(D + J dtau_k - E_k + Y_k/mu_k)        (Eq. update_A, cf. Eq. A_1)
        E_{k+1}   = argmin_E L = T_{lam/mu_k}(D + J dtau_k - A_{k+1} + Y_k/mu_k)  (Eq. update_E, cf. Eq. E_1)
        dtau_{k+1} = argmin_dtau L = G^{-1} J^T (A_{k+1} + E_{k+1} - D - Y_k/mu_k) (Eq. update_detla_Tau;
                     with the constraint rows Q the stacked least squares of P:671-684: G = J^TJ + Q^TQ)
        Y_{k+1}   = Y_k + mu_k (D + J dtau_{k+1} - A_{k+1} - E_{k+1})
        mu_{k+1}  = rho mu_k  (unbounded)
    initialised A_0 = D, E_0 = 0, Y_0 = 0, dtau_0 = 0. Stops when the constraint
    residual ||D + J dtau - A - E||_F/||D||_F < tol (reading Z24) unless ``fixed_iters`` > 0.
    """
    a, e, y = dh.copy(), np.zeros_like(dh), np.zeros_like(dh)
    dtau = np.zeros(proj.jm.shape[1])
    jdt = np.zeros_like(dh)
    nd = float(np.linalg.norm(dh)) or 1.0
    mu = mu0
    n_iter = fixed_iters if fixed_iters > 0 else max_inner
    sig = None
    resid = float("nan")
    for k in range(n_iter):
        a, sig = svt(dh + jdt - e + y / mu, 1.0 / mu)
        e = shrink(dh + jdt - a + y / mu, lam / mu)
        dtau = proj.delta_tau(a + e - dh - y / mu)
        jdt = (proj.jm @ dtau).reshape(dh.shape)
        r = dh + jdt - a - e
        y = y + mu * r
        resid = float(np.linalg.norm(r)) / nd
        mu_used = mu
        mu = rho * mu
        if resid < tol and fixed_iters <= 0:
            return AdmResult(a, e, y, dtau, k + 1, mu_used, sig, resid, True)
    return AdmResult(a, e, y, dtau, n_iter, mu / rho, sig, resid, resid < tol)


# ----------------------------------------------------------------------------------------------
# Algorithm 1: TILT via LADMAP + VWS
# ----------------------------------------------------------------------------------------------

def relative_rank(sigma_a):
    """Reading Z19: rank = #{sigma_j(A) > 1e-3 sigma_1(A)}; band flag if a ratio is in [3e-4, 3e-3]."""
    s = np.sort(np.asarray(sigma_a, dtype=np.float64))[::-1]
    if s.size == 0 or s[0] <= 0:
        return 0, False
    ratio = s / s[0]
    return int(np.sum(ratio > 1e-3)), bool(np.any((ratio >= 3e-4) & (ratio <= 3e-3)))


def tilt(image, box, tau0, kind, prm: Params = Params(), rho_replay=None, warm=None, inner_replay=None):
    """Algorithm 1 for one window; returns a dict (tau, A, E, Y, report fields, traces).

    Step 1: normalise D o tau and compute J; Q per reading Z10.
    Step 2: LADMAP with the warm starts A_0 = A_inf, E_0 = E_inf (Eq. warm_start) and
            Y_0 = W^TW Y_inf (Eq. Y_new_warmstart); first pass A_0 = D o tau, E_0 = Y_0 = 0
            (reading Z4). mu_0 = mu0_scale/sigma_1(D_hat) each inner loop (Z3, Z5).
    Step 3: Delta tau* (Eq. Delta_tau; with Q the stacked least squares P:671-684).
    Step 4: tau^{i+1} = tau^i + Delta tau* (P:568-570).
    Outer stop ("while not converged", reading Z9).
    ``rho_replay``: optional list (per outer iteration) of 0/1 sequences (reading Z21).
    ``inner_replay``: optional list (per outer iteration) of inner-iteration counts: the inner loop
    of outer iteration i runs exactly inner_replay[i] iterations (replaying another run's Cond1 &
    Cond2 decisions; parity protocol, reading Z21).
    ``warm``: optional (A, E, Y) that replace the first inner loop's cold start A_0 = D_hat,
    E_0 = Y_0 = 0 (then Y_0 <- W^TW Y as every warm start, Eq. Y_new_warmstart); used by
    the pyramid's fine level (reading Z26). Ignored without VWS.
    """
    m, n = int(box[3]), int(box[2])
    lam = prm.lam if prm.lam > 0 else 1.0 / math.sqrt(max(m, n))
    tau = np.asarray(tau0, dtype=np.float64).copy()
    a = e = y = None
    if warm is not None and prm.vws:
        a, e, y = (np.asarray(x, dtype=np.float64).copy() for x in warm)
    f_prev = None
    status = MAX_OUTER
    stop_rule = STOP_NONE
    outer_traces = []
    tau_path = []       # tau after every outer iteration (test instrumentation)
    inner_iters = 0
    res = None
    nd = float("nan")
    dtau_inf = float("nan")
    f = float("nan")
    n_outer = prm.fixed_outer_iters if prm.fixed_outer_iters > 0 else prm.max_outer
    it_done = 0
    for it in range(n_outer):
        d, jraw, st = warp(image, box, tau, kind)
        if st != CONVERGED:
            status = st
            break
        nd = float(np.linalg.norm(d))
        if nd == 0.0:
            status = ZERO_PATCH
            break
        dh, j, nd = normalise(d, jraw)
        q = constraints_q(tau, kind, m, n) if prm.constraints else None
        try:
            proj = Projector(j, q)
        except Projector.SingularGram:
            status = SINGULAR_GRAM
            break
        sigma1 = float(np.linalg.svd(dh, compute_uv=False)[0])
        mu0 = prm.mu0_scale / sigma1
        if prm.inner == "adm":
            # the original method: cold start every outer iteration, dtau from the ADM
            res = adm(dh, proj, lam, mu0, prm.adm_rho, prm.adm_tol, prm.max_inner, fixed_iters=prm.fixed_inner_iters)
            a, e, y = res.A, res.E, res.Y
            inner_iters += res.iters
            outer_traces.append([])
            dtau = res.dtau
        else:
            if a is None or not prm.vws:
                a, e, y = dh.copy(), np.zeros_like(dh), np.zeros_like(dh)
            else:
                y = proj.apply(y)                      # Eq. Y_new_warmstart
            replay = rho_replay[it] if rho_replay is not None and it < len(rho_replay) else None
            noise = ((prm.crit_noise, np.random.default_rng([prm.noise_seed, it]))
                     if prm.crit_noise > 0 else None)
            fixed = prm.fixed_inner_iters
            if inner_replay is not None and it < len(inner_replay):
                fixed = int(inner_replay[it])
            res = ladmap(dh, proj, lam, mu0, prm.mu_max_ratio * mu0, prm.rho0, prm.eps1, prm.eps2,
                         prm.max_inner, a, e, y, fixed_iters=fixed, rho_replay=replay, svd=prm.svd,
                         crit_noise=noise)
            a, e, y = res.A, res.E, res.Y
            inner_iters += res.iters
            outer_traces.append(res.trace)
            dtau = proj.delta_tau(a + e - dh)          # Step 3
        tau = tau + dtau                           # Step 4
        if prm.tau_noise > 0:
            tau = tau * (1.0 + prm.tau_noise * np.random.default_rng([prm.noise_seed, 7, it]).standard_normal(tau.shape))
        tau_path.append(tau.copy())
        dtau_inf = float(np.max(np.abs(dtau)))
        f = float(shrink(res.sigma_m, 1.0 / res.mu).sum()) + lam * float(np.abs(e).sum())
        it_done = it + 1
        if not np.isfinite(f) or f > 1e12 or not np.all(np.isfinite(tau)):
            status = DIVERGED
            break
        rule = STOP_NONE
        if f_prev is not None and abs(f - f_prev) < prm.obj_tol * abs(f_prev):
            rule = STOP_OBJECTIVE
        elif dtau_inf < prm.tau_tol:
            rule = STOP_DTAU
        f_prev = f
        if rule != STOP_NONE:
            status, stop_rule = CONVERGED, rule
            if prm.fixed_outer_iters <= 0:
                break
        else:
            status, stop_rule = MAX_OUTER, STOP_MAX_OUTER
    sig_a = shrink(res.sigma_m, 1.0 / res.mu) if res is not None else np.zeros(1)
    rank, band = relative_rank(sig_a)
    return {
        "status": status, "stop_rule": stop_rule, "tau": tau, "A": a, "E": e, "Y": y,
        "outer_iters": it_done, "inner_iters": inner_iters, "objective": f,
        "rank": rank, "rank_band": band, "svt_rank": int(np.sum(res.sigma_m > 1.0 / res.mu)) if res else 0,
        "crit1": (res.resid if isinstance(res, AdmResult) else res.crit1) if res else float("nan"),
        "crit2": (float("nan") if isinstance(res, AdmResult) else res.crit2) if res else float("nan"),
        "patch_norm": nd, "dtau_inf": dtau_inf, "traces": outer_traces, "lam": lam, "tau_path": tau_path,
    }


def downsample2x(image):
    """2x2 box filter for the 2-level pyramid of config 3 (reading Z18; the paper has none)."""
    img = np.asarray(image, dtype=np.float64)
    hh, ww = img.shape[0] // 2 * 2, img.shape[1] // 2 * 2
    img = img[:hh, :ww]
    return 0.25 * (img[0::2, 0::2] + img[0::2, 1::2] + img[1::2, 0::2] + img[1::2, 1::2])


def upsample2x_warm(x):
    """Coarse-level state -> fine-level warm start (reading Z26): 2x2 replication, halved. The
    coarse and fine D_hat are both unit-norm and replication doubles the Frobenius and spectral
    norms, so up(X)/2 keeps ||.||_F and ||.||_2 (the dual's ||Y||_2 <= 1 and, as lambda_f =
    lambda_c/sqrt(2) >= lambda_c/2, ||Y||_inf <= lambda_f stay feasible)."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * np.repeat(np.repeat(x, 2, axis=0), 2, axis=1)


def tilt_pyramid(image, box, tau0, kind, prm: Params = Params(), levels: int = 2):
    """Coarse-to-fine TILT (reading Z18): solve on the 2x2-downsampled image with box/2, then on the
    full image starting from the coarse tau (unchanged: the normalised frames coincide); with
    ``prm.pyramid_warm`` the fine level's first inner loop also starts from the coarse A, E, Y
    (upsample2x_warm, reading Z26) when the coarse level produced them."""
    if levels <= 1:
        return tilt(image, box, tau0, kind, prm)
    coarse_img = np.asarray(image, dtype=np.float64)
    x0, y0, w, h = (int(v) for v in box)
    for _ in range(levels - 1):
        coarse_img = downsample2x(coarse_img)
        x0, y0, w, h = x0 // 2, y0 // 2, w // 2, h // 2
    res_c = tilt(coarse_img.astype(np.float32).astype(np.float64), (x0, y0, w, h), tau0, kind,
                 replace(prm, lam=prm.lam))
    # the fine level always starts from the coarse tau (a failed coarse level keeps its last tau)
    warm = None
    if prm.pyramid_warm and levels == 2 and res_c["status"] in (CONVERGED, MAX_OUTER) and res_c["A"] is not None:
        warm = tuple(upsample2x_warm(res_c[k]) for k in ("A", "E", "Y"))
    res_f = tilt(image, box, res_c["tau"], kind, prm, warm=warm)
    for key in ("outer_iters", "inner_iters"):
        res_f[key] += res_c[key]
    res_f["coarse"] = res_c
    return res_f


def _tilt_job(args):
    image, box, tau0, kind, prm, levels = args
    return tilt_pyramid(image, box, tau0, kind, prm, levels)


def tilt_batch(images, patch_image, boxes, tau0, kind, prm: Params = Params(), levels=1,
               n_workers=1):
    """Independent patches (north_star: "large batches of independent image patches")."""
    jobs = [(np.asarray(images[patch_image[b]], dtype=np.float64), boxes[b], tau0[b], kind, prm, levels)
            for b in range(len(boxes))]
    if n_workers <= 1 or len(jobs) <= 1:
        return [_tilt_job(j) for j in jobs]
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(min(n_workers, len(jobs))) as pool:
        return pool.map(_tilt_job, jobs)


def tilt_oracle_solve_batch(images, n_images, H, W, patch_image, boxes, tau0, B, kind, prm: Params = Params(),
                            n_threads=1, levels=1):
    """The oracle twin of tilt_solve_batch: the same argument meaning on host fp64
    arrays -- images [n_images][H][W], patch_image [B], boxes [B][4] = (x0, y0, w, h), tau0 [B][p] or
    None (identity), kind AFFINE / HOMOGRAPHY -- plus n_threads worker processes. Returns (tau [B][p],
    A [B][m][n], E [B][m][n], reports: list of dicts with status, stop_rule, outer_iters, inner_iters,
    objective, rank, crit1, crit2, patch_norm). A patch without a state (window escape, singular Gram
    or zero patch in its first outer iteration) gets zero A and E, as the C ABI."""
    images = np.asarray(images, dtype=np.float64).reshape(n_images, H, W)
    boxes = np.asarray(boxes, dtype=np.int64).reshape(B, 4)
    p = 8 if kind == HOMOGRAPHY else 6
    if tau0 is None:
        t0 = np.zeros((B, p))
        t0[:, 0] = 1.0
        t0[:, 3] = 1.0
    else:
        t0 = np.asarray(tau0, dtype=np.float64).reshape(B, p)
    res = tilt_batch(images, np.asarray(patch_image).reshape(B), boxes, t0, kind, prm, levels=levels,
                     n_workers=n_threads)
    m, n = (int(boxes[0, 3]), int(boxes[0, 2])) if B > 0 else (0, 0)
    tau = np.stack([r["tau"] for r in res]) if B > 0 else np.zeros((0, p))
    A = np.stack([r["A"] if r["A"] is not None else np.zeros((m, n)) for r in res]) if B > 0 else np.zeros((0, m, n))
    E = np.stack([r["E"] if r["E"] is not None else np.zeros((m, n)) for r in res]) if B > 0 else np.zeros((0, m, n))
    keys = ("status", "stop_rule", "outer_iters", "inner_iters", "objective", "rank", "crit1", "crit2", "patch_norm")
    reps = [{k: r[k] for k in keys} for r in res]
    return tau, A, E, reps
