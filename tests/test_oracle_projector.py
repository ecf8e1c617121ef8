"""Pins for the oracle projector and Delta tau.

The oracle implements W^TW = I - J (J^TJ + Q^TQ)^{-1} J^T implicitly (Eq. Jperpv). These tests
check it against the paper's *other* statements: J_perp symmetric and idempotent (Eq.
J_properties), ||J_perp|| = 1 (Prop. 2), the explicit W of P:693-698 whose
product W^TW must equal the operator (Eq. WTW_property) and ||W||_2 = 1, and
Delta tau as the least-squares solution of the stacked system via numpy lstsq.
"""
import numpy as np
import pytest

import oracle as O


def _dense(proj, mn):
    cols = []
    for k in range(mn):
        e = np.zeros(mn)
        e[k] = 1.0
        cols.append(proj.apply(e.reshape(proj.shape)).reshape(-1))
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("seed", range(5))
def test_jperp_properties(seed):
    rng = np.random.default_rng(seed)
    m, n, p = 5, 8, 3
    j = rng.normal(size=(p, m, n))
    proj = O.Projector(j)
    pd = _dense(proj, m * n)
    np.testing.assert_allclose(pd, pd.T, atol=1e-10)            # symmetric
    np.testing.assert_allclose(pd @ pd, pd, atol=1e-10)          # idempotent
    ev = np.linalg.eigvalsh(0.5 * (pd + pd.T))
    assert np.all(np.minimum(np.abs(ev), np.abs(ev - 1)) < 1e-8)  # eigenvalues in {0, 1}
    assert np.sum(ev > 0.5) == m * n - p
    # ||J_perp|| = 1 by power iteration (Prop. 2)
    x = rng.normal(size=m * n)
    for _ in range(50):
        x = pd @ x
        x /= np.linalg.norm(x)
    assert np.linalg.norm(pd @ x) == pytest.approx(1.0, abs=1e-8)
    # annihilates span(J), fixes its complement
    w = rng.normal(size=p)
    jw = np.tensordot(w, j, axes=1)
    assert np.linalg.norm(proj.apply(jw)) < 1e-10 * np.linalg.norm(jw)
    v = rng.normal(size=(m, n))
    v_perp = proj.apply(v)
    np.testing.assert_allclose(proj.apply(v_perp), v_perp, atol=1e-10)


def test_jperp_trivial_example():
    # J = (1, 0)^T -> J_perp = [[0, 0], [0, 1]]
    proj = O.Projector(np.array([[[1.0, 0.0]]]))
    np.testing.assert_allclose(_dense(proj, 2), [[0, 0], [0, 1]], atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_wtw_identity_against_explicit_w(seed):
    rng = np.random.default_rng(100 + seed)
    m, n, p, l = 5, 8, 4, 2
    j = rng.normal(size=(p, m, n))
    q = rng.normal(size=(l, p))
    proj = O.Projector(j, q)
    jm = j.reshape(p, -1).T
    ginv = np.linalg.inv(jm.T @ jm + q.T @ q)
    w = np.vstack([np.eye(m * n) - jm @ ginv @ jm.T, -q @ ginv @ jm.T])
    np.testing.assert_allclose(w.T @ w, _dense(proj, m * n), atol=1e-10)  # Eq. WTW_property
    assert np.linalg.norm(w, 2) == pytest.approx(1.0, abs=1e-8)           # ||W||_2 = 1
    # Q = 0 rows reduce W^TW to J_perp exactly
    np.testing.assert_allclose(_dense(O.Projector(j, np.zeros((1, p))), m * n),
                               _dense(O.Projector(j), m * n), atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_delta_tau(seed):
    rng = np.random.default_rng(200 + seed)
    m, n, p = 6, 7, 5
    j = rng.normal(size=(p, m, n))
    wtrue = rng.normal(size=p)
    r = np.tensordot(wtrue, j, axes=1)
    # A + E - D = J w with Q absent -> Delta tau = w
    np.testing.assert_allclose(O.Projector(j).delta_tau(r), wtrue, atol=1e-10)
    # A + E = D -> 0
    np.testing.assert_allclose(O.Projector(j).delta_tau(np.zeros((m, n))), 0.0, atol=0)
    # with Q: least-squares solution of [J; Q] dtau = [r; 0]
    q = rng.normal(size=(3, p))
    rr = rng.normal(size=(m, n))
    stacked = np.vstack([j.reshape(p, -1).T, q])
    rhs = np.concatenate([rr.reshape(-1), np.zeros(3)])
    ls = np.linalg.lstsq(stacked, rhs, rcond=None)[0]
    np.testing.assert_allclose(O.Projector(j, q).delta_tau(rr), ls, atol=1e-9)


def test_singular_gram_detected():
    j = np.zeros((4, 3, 3))
    with pytest.raises(O.Projector.SingularGram):
        O.Projector(j)
