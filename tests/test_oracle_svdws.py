"""Pins for the oracle's SVD warm start (Algorithm 2; Appendix A; SURVEY.md
NEXT-1 / P15). Independent of the formulas being tested: central finite differences of
f(t) = 1/2 ||M - U(t) Sigma(t) V(t)^T||^2 along the Cayley curve (pins f'(0), f''(0) and thereby
h''(0) = -P_U Z + Z P_V), the Cayley properties of P:810-816, the descent the Taylor step is built
for, and the paper's pseudocontraction bound on the resulting SVT."""
import numpy as np
import pytest

import oracle as O
import tilt_synth as ts


def _case(m, n, delta, seed):
    rng = np.random.default_rng(seed)
    m0 = rng.normal(size=(m, n))
    u, s, vt = np.linalg.svd(m0, full_matrices=False)
    return m0, m0 + delta * rng.normal(size=(m, n)), u, s, vt.T


def _derivs(m1, u, s, v):
    w = (u * s) @ v.T
    pu = w @ m1.T - m1 @ w.T
    pv = w.T @ m1 - m1.T @ w
    ps = s - np.einsum("ij,ij->j", u, m1 @ v)
    h0 = m1 - w
    ups = (u * ps) @ v.T
    h1 = pu @ w + ups - w @ pv
    z = h1 + ups
    h2 = -pu @ z + z @ pv
    return float(np.sum(h0 * h1)), float(np.sum(h1 * h1) + np.sum(h0 * h2)), pu, pv


@pytest.mark.parametrize("m,n,delta,seed", [(12, 9, 1e-2, 0), (20, 20, 3e-2, 1), (30, 7, 1e-1, 2)])
def test_appendix_a_derivatives_match_finite_differences(m, n, delta, seed):
    m0, m1, u, s, v = _case(m, n, delta, seed)
    f1, f2, pu, pv = _derivs(m1, u, s, v)
    f = lambda t: O.cayley_objective(m1, u, s, v, t)  # noqa: E731
    h = 1e-4 / max(1.0, np.linalg.norm(pu))
    fd1 = (f(h) - f(-h)) / (2 * h)
    fd2 = (f(h) - 2 * f(0.0) + f(-h)) / h ** 2
    assert f1 == pytest.approx(fd1, rel=1e-6, abs=1e-12)
    assert f2 == pytest.approx(fd2, rel=1e-4)
    # P_U, P_V are skew (tangent directions of the Stiefel manifolds)
    assert np.abs(pu + pu.T).max() < 1e-12 and np.abs(pv + pv.T).max() < 1e-12


@pytest.mark.parametrize("m,n,delta,seed", [(12, 9, 1e-2, 0), (20, 20, 3e-2, 1), (30, 7, 1e-1, 2)])
def test_taylor_step_properties(m, n, delta, seed):
    m0, m1, u, s, v = _case(m, n, delta, seed)
    ut, st, vt, t = O.svd_warm_start(m1, u, s, v)
    # Cayley properties 2 (feasibility) of P:810-816
    assert np.abs(ut.T @ ut - np.eye(n)).max() < 1e-12
    assert np.abs(vt.T @ vt - np.eye(n)).max() < 1e-12
    # the step descends f (t* minimises the quadratic model, f''(0) > 0 here)
    assert O.cayley_objective(m1, u, s, v, t) < O.cayley_objective(m1, u, s, v, 0.0)
    # ||S_eps(U Sigma V^T (t*)) - S_eps(M_k)|| <= ||approx - M_k|| <= ||M_{k-1} - M_k||
    for eps in (0.05, 0.3, 1.0):
        approx = (ut * O.shrink(st, eps)) @ vt.T
        exact = O.svt(m1, eps)[0]
        err = np.linalg.norm(approx - exact)
        assert err <= np.linalg.norm((ut * st) @ vt.T - m1) + 1e-12
        assert err <= np.linalg.norm(m1 - m0) + 1e-12


def test_exact_previous_svd_is_a_fixed_point():
    m0, _, u, s, v = _case(10, 6, 0.0, 3)
    ut, st, vt, t = O.svd_warm_start(m0, u, s, v)
    # gradients vanish to rounding, so whatever t* the 0/0 ratio gives, the SVD does not move
    np.testing.assert_allclose((ut * st) @ vt.T, m0, atol=1e-12)
    np.testing.assert_allclose(st, s, atol=1e-12)


def test_ladmap_svdws_tight_gate_keeps_ladmap_iterations():
    """LADMAP+SVDWS (Table 1's third column): with the gate at 2e-5 ||D||_F the warm step
    is taken on some iterations and the iteration count and objective stay LADMAP's (the paper:
    'the SVD warm start only changes the number of iterations very slightly')."""
    its, its_w, rel, warm = [], [], [], 0
    for s in range(5):
        inst = ts.table1_instance(10, 6, s)
        proj = O.Projector(inst["J"])
        mu0 = 1.25 / np.linalg.svd(inst["D"], compute_uv=False)[0]
        z = np.zeros_like(inst["D"])
        args = (inst["D"], proj, inst["lam"], mu0, 1e6 * mu0, 2.0, 1e-6, 0.1, 1000, inst["D"].copy(), z, z)
        r0 = O.ladmap(*args)
        sw = O.SvdWarm(2e-5 * np.linalg.norm(inst["D"]))
        r1 = O.ladmap(*args, svd=sw)
        warm += sw.warm_steps
        its.append(r0.iters)
        its_w.append(r1.iters)
        rel.append(abs(O.objective(r1.A, r1.E, inst["lam"]) / O.objective(r0.A, r0.E, inst["lam"]) - 1))
    assert warm > 0
    assert abs(np.mean(its_w) - np.mean(its)) <= 3
    assert max(rel) < 1e-4


def test_svdws_step_rule_is_the_quadratic_model_only():
    """Reading Z27 (Eq. ft): with the gate open, the warm step is taken exactly when the
    quadratic model has a minimiser (f''(0) > 0, computed here by this file's own Appendix A
    derivatives), however large (t*/2) P is -- the Cayley curve is feasible for every t,
    so the step must come back with orthonormal U and orthogonal V; f''(0) <= 0 takes a full SVD,
    whose S_eps is then exact."""
    taken = rejected = 0
    big_steps = 0
    for seed in range(40):
        rng = np.random.default_rng([77, seed])
        m0 = rng.normal(size=(12, 10))
        m1 = rng.normal(size=(12, 10)) * rng.uniform(0.1, 3.0)
        sw = O.SvdWarm(1e9)                 # the gate never closes
        sw.svt(m0, 0.1)                     # first call: full SVD
        u, s, vt = np.linalg.svd(m0, full_matrices=False)
        f1, f2, pu, pv = _derivs(m1, u, s, vt.T)
        a1, _ = sw.svt(m1, 0.1)
        assert sw.decisions == [0, 1 if f2 > 0 else 0]
        if f2 > 0:
            taken += 1
            ut, st, vv = sw.prev
            t = -f1 / f2
            big_steps += max(np.linalg.norm(0.5 * t * pu), np.linalg.norm(0.5 * t * pv)) >= 0.5
            assert np.abs(ut.T @ ut - np.eye(10)).max() < 1e-10
            assert np.abs(vv.T @ vv - np.eye(10)).max() < 1e-10
        else:
            rejected += 1
            np.testing.assert_allclose(a1, O.svt(m1, 0.1)[0], atol=1e-12)
    assert taken > 0 and rejected > 0 and big_steps > 0
