"""Pins for the oracle's proximal operators and SVD step.

Each check is tied to something other than the oracle's own formula: closed forms printed in the
paper / SPEC examples, a brute-force grid minimiser, an independent eigen-solver, the subgradient
characterisation of the nuclear-norm prox, and the paper's pseudocontraction inequality.
"""
import numpy as np
import pytest

import oracle as O


def test_shrink_closed_form():
    # P:482 T_eps(x) = sgn(x) max(|x| - eps, 0); SPEC S:56-57 examples
    assert O.shrink(1.2, 0.5) == pytest.approx(0.7)
    assert O.shrink(-0.3, 0.5) == 0.0
    assert O.shrink(-2.0, 0.5) == pytest.approx(-1.5)
    assert O.shrink(0.5, 0.5) == 0.0


def test_shrink_is_argmin_grid():
    # T_{lam/mu}(x) = argmin_e lam|e| + mu/2 (e - x)^2  (Eq. E P:444 / Eq. E_1), brute force
    rng = np.random.default_rng(0)
    lam, mu = 0.3, 2.0
    grid = np.arange(-3.0, 3.0, 1e-4)
    for x in rng.uniform(-2, 2, size=20):
        f = lam * np.abs(grid) + 0.5 * mu * (grid - x) ** 2
        assert O.shrink(x, lam / mu) == pytest.approx(grid[np.argmin(f)], abs=2e-4)


def test_svt_closed_forms():
    # diag(3,1), eps=2 -> diag(1,0); eps = 0 -> M
    a, sig = O.svt(np.diag([3.0, 1.0]), 2.0)
    np.testing.assert_allclose(a, np.diag([1.0, 0.0]), atol=1e-14)
    rng = np.random.default_rng(1)
    m = rng.normal(size=(7, 5))
    np.testing.assert_allclose(O.svt(m, 0.0)[0], m, atol=1e-12)
    # eps above sigma_1 kills everything
    np.testing.assert_allclose(O.svt(m, 1e3)[0], 0.0, atol=0)


@pytest.mark.parametrize("shape", [(6, 6), (9, 5), (5, 9), (30, 30)])
def test_svt_subgradient_certificate(shape):
    """A = S_eps(M) iff M - A in eps * d||A||_*, i.e. ||M - A||_2 <= eps and <M - A, A> = eps ||A||_*
    (prox of the nuclear norm). Norms via an independent symmetric eigensolver."""
    rng = np.random.default_rng(shape[0] * 31 + shape[1])
    m = rng.normal(size=shape)
    eps = 0.7 * np.linalg.norm(m, 2) / 3
    a, _ = O.svt(m, eps)
    r = m - a
    spec = np.sqrt(np.max(np.linalg.eigvalsh(r.T @ r)))
    ev = np.linalg.eigvalsh(a.T @ a)
    nuc = np.sum(np.sqrt(ev[ev > 1e-12 * ev.max()]))
    assert spec <= eps * (1 + 1e-12)
    assert np.sum(r * a) == pytest.approx(eps * nuc, rel=1e-10)
    # and it beats random perturbations on eps||A||_* + 1/2||A - M||^2
    def obj(x):
        return eps * np.sum(np.linalg.svd(x, compute_uv=False)) + 0.5 * np.sum((x - m) ** 2)
    f0 = obj(a)
    for _ in range(10):
        assert obj(a + 1e-3 * rng.normal(size=shape)) >= f0


@pytest.mark.parametrize("k", range(1, 9))
def test_svd_step_reconstruction_tiny(k):
    # P3: reconstruction / orthogonality on tiny matrices incl. rank-deficient and repeated sigma
    rng = np.random.default_rng(k)
    mats = [rng.normal(size=(k, k)), np.eye(k) * 2.0, np.outer(rng.normal(size=k), rng.normal(size=k))]
    for mm in mats:
        u, s, vt = np.linalg.svd(mm)
        assert np.linalg.norm(mm - (u * s) @ vt) <= 1e-12 * max(1.0, np.linalg.norm(mm))
        assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-12
        assert np.linalg.norm(vt @ vt.T - np.eye(k)) <= 1e-12
        # sigma^2 vs an independent symmetric eigensolver of M^T M
        np.testing.assert_allclose(np.sort(s ** 2), np.sort(np.linalg.eigvalsh(mm.T @ mm)), atol=1e-8)
    _, sig = O.svt(np.eye(3), 0.0)
    np.testing.assert_allclose(sig, [1, 1, 1])


def test_pseudocontraction_inequality():
    """||S(W1)-S(W2)||^2 <= ||W1-W2||^2 - ||(S(W1)-W1)-(S(W2)-W2)||^2 (and for T_eps)."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        w1, w2 = rng.normal(size=(2, 8, 6))
        eps = rng.uniform(0.1, 2.0)
        s1, s2 = O.svt(w1, eps)[0], O.svt(w2, eps)[0]
        lhs = np.sum((s1 - s2) ** 2)
        rhs = np.sum((w1 - w2) ** 2) - np.sum(((s1 - w1) - (s2 - w2)) ** 2)
        assert lhs <= rhs + 1e-8
        t1, t2 = O.shrink(w1, eps), O.shrink(w2, eps)
        assert np.sum((t1 - t2) ** 2) <= np.sum((w1 - w2) ** 2) - np.sum(((t1 - w1) - (t2 - w2)) ** 2) + 1e-8


def test_objective_closed_forms():
    # A = diag(2,3), E = 0 -> 5; A = 0, k entries +-1, lam = .5 -> .5k
    assert O.objective(np.diag([2.0, 3.0]), np.zeros((2, 2)), 1.0) == pytest.approx(5.0)
    e = np.zeros((4, 4))
    e[0, 0], e[1, 2], e[3, 3] = 1, -1, 1
    assert O.objective(np.zeros((4, 4)), e, 0.5) == pytest.approx(1.5)


# ---------------------------------------------------------------------------------------------
# The oracle's own one-sided Jacobi SVD (SURVEY.md §8(c) oracle step 5, P3)
# ---------------------------------------------------------------------------------------------
def _tiny_cases():
    rng = np.random.default_rng(7)
    cases = [np.eye(3), np.array([[2.0]]), np.zeros((3, 2)), np.diag([3.0, 3.0, 1.0])]  # repeated sigma
    for (m, n) in [(1, 4), (4, 1), (2, 2), (3, 5), (5, 3), (8, 8)]:
        cases.append(rng.normal(size=(m, n)))
    u = rng.normal(size=(6, 2))
    cases.append(u @ rng.normal(size=(2, 7)))  # rank 2 of 6 x 7
    q, _ = np.linalg.qr(rng.normal(size=(5, 5)))
    cases.append(q @ np.diag([2.0, 2.0, 2.0, 1e-9, 0.0]) @ q.T)  # repeated + near-zero + zero
    return cases


@pytest.mark.parametrize("k", range(12))
def test_jacobi_svd_reconstruction_orthogonality(k):
    w = _tiny_cases()[k]
    u, s, v, sweeps = O.jacobi_svd(w)
    scale = max(np.linalg.norm(w), 1.0)
    assert np.linalg.norm(u * s @ v.T - w) <= 1e-12 * scale
    assert np.linalg.norm(v.T @ v - np.eye(w.shape[1])) <= 1e-12
    keep = s > 1e-9 * max(s.max(), 1e-300)
    uk = u[:, keep]
    assert np.linalg.norm(uk.T @ uk - np.eye(int(keep.sum()))) <= 1e-10
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0) and sweeps <= 60


def test_jacobi_svd_identity_and_eigen():
    # I_3 -> sigma = (1, 1, 1) with no rotation
    _, s, _, sweeps = O.jacobi_svd(np.eye(3))
    np.testing.assert_array_equal(s, [1.0, 1.0, 1.0])
    assert sweeps == 1
    # sigma^2 against an independent symmetric eigen-solver of M^T M (not the library SVD)
    rng = np.random.default_rng(3)
    for (m, n) in [(9, 6), (6, 9), (12, 12)]:
        w = rng.normal(size=(m, n))
        s = O.jacobi_svd(w)[1]
        ev = np.sort(np.linalg.eigvalsh(w.T @ w))[::-1][:min(m, n)]
        np.testing.assert_allclose(s[:min(m, n)] ** 2, ev, rtol=1e-9, atol=1e-10)


def test_jacobi_svt_equals_library_svt_and_warm_start():
    rng = np.random.default_rng(4)
    w = rng.normal(size=(20, 16)) @ np.diag(np.linspace(3, 0.01, 16))
    for eps in (0.0, 0.05, 0.7, 5.0):
        a_j, s_j = O.svt(w, eps, "jacobi")
        a_l, s_l = O.svt(w, eps, "lapack")
        np.testing.assert_allclose(a_j, a_l, atol=1e-12 * np.linalg.norm(w))
        np.testing.assert_allclose(s_j, s_l, atol=1e-12 * s_l[0])
    # warm start from the right vectors of a nearby matrix: same SVD, fewer sweeps
    _, _, v, cold = O.jacobi_svd(w)
    w2 = w + 1e-4 * rng.normal(size=w.shape)
    u2, s2, v2, warm = O.jacobi_svd(w2, v0=v)
    assert warm < O.jacobi_svd(w2)[3]
    np.testing.assert_allclose(u2 * s2 @ v2.T, w2, atol=1e-12 * np.linalg.norm(w2))


def test_ladmap_same_with_own_jacobi_svd():
    """A fixed count of LADMAP iterations with the oracle's Jacobi SVD equals the library-SVD run."""
    import tilt_synth as ts
    inst = ts.table1_instance(10, 6, 0)
    proj = O.Projector(inst["J"])
    mu0 = 1.25 / np.linalg.svd(inst["D"], compute_uv=False)[0]
    z = np.zeros_like(inst["D"])
    runs = [O.ladmap(inst["D"], proj, inst["lam"], mu0, 1e6 * mu0, 2.0, 1e-6, 0.1, 15, inst["D"].copy(), z, z,
                     fixed_iters=15, svd=m) for m in ("lapack", "jacobi")]
    np.testing.assert_allclose(runs[1].A, runs[0].A, atol=1e-10)
    np.testing.assert_allclose(runs[1].E, runs[0].E, atol=1e-10)
