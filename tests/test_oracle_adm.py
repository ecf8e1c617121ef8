"""Pins for the oracle's ADM baseline inner loop, independent of its
own formula: the iteration counts and objectives the paper prints in Table 1 (statistical pin,
tests/golden/table1.json), Proposition 1 (ADM with a slowly growing penalty and LADMAP reach the same
optimum of the same convex program), the exact stationarity of the dtau step
(J^T Y_k = 0), and dual feasibility of the converged multiplier (P:639-652 with erratum E3)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import tilt_synth as ts

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))


def _run_adm(inst, rho=1.25, tol=1e-7, max_inner=500, fixed=0):  # 1e-7: Table 1's regime (Z24)
    proj = O.Projector(inst["J"])
    mu0 = 1.25 / np.linalg.svd(inst["D"], compute_uv=False)[0]
    return O.adm(inst["D"], proj, inst["lam"], mu0, rho, tol, max_inner, fixed_iters=fixed), proj, mu0


@pytest.mark.parametrize("row", GOLD["adm_rows"][:2], ids=lambda r: f"n{r['size']}")
def test_table1_adm_iterations_and_objective(row):
    n = row["size"]
    its, objs = [], []
    for s in range(10):
        inst = ts.table1_instance(n, 6, s)
        r, _, _ = _run_adm(inst)
        assert r.converged
        its.append(r.iters)
        objs.append(O.objective(r.A, r.E, inst["lam"]))
    assert abs(np.mean(its) - row["iters"]) <= 3.0, np.mean(its)
    # Table 1's LADMAP objectives are matched within 2% by the oracle (test_oracle_inner); the ADM
    # stops at a slightly worse point (the paper: ADM "may produce an incorrect solution")
    assert np.mean(objs) == pytest.approx(row["objective"], rel=0.03)


def test_table1_adm_needs_more_iterations_than_ladmap():
    """Table 1: LADMAP uses less than half of ADM's iterations."""
    for s in range(4):
        inst = ts.table1_instance(50, 6, s)
        r, proj, mu0 = _run_adm(inst)
        z = np.zeros_like(inst["D"])
        lr = O.ladmap(inst["D"], proj, inst["lam"], mu0, 1e6 * mu0, 2.0, 1e-6, 0.1, 1000, inst["D"].copy(), z, z)
        assert lr.iters < 0.6 * r.iters, (lr.iters, r.iters)


def test_adm_dtau_step_stationarity_and_mu_schedule():
    inst = ts.table1_instance(12, 6, 3)
    jm = inst["J"].reshape(6, -1).T
    for k in (1, 2, 5, 17):
        r, _, mu0 = _run_adm(inst, fixed=k)
        # dtau minimises L exactly: J^T Y_{k+1} = 0 (no constraint rows)
        assert np.linalg.norm(jm.T @ r.Y.reshape(-1)) <= 1e-9 * max(1.0, np.linalg.norm(r.Y))
        assert r.mu == pytest.approx(mu0 * 1.25 ** (k - 1), rel=1e-12)


def test_adm_slow_penalty_reaches_ladmap_optimum():
    """Proposition 1: the 3-variable problem (ADM) and the 2-variable reformulation
    (LADMAP) have the same optimum; a slowly growing penalty ADM converges to it."""
    for s in range(3):
        inst = ts.table1_instance(8, 4, s)
        r, proj, mu0 = _run_adm(inst, rho=1.02, tol=1e-11, max_inner=5000)
        z = np.zeros_like(inst["D"])
        lr = O.ladmap(inst["D"], proj, inst["lam"], mu0, 1e8 * mu0, 1.1, 1e-11, 1e-7, 20000, inst["D"].copy(), z, z)
        fa = O.objective(r.A, r.E, inst["lam"])
        fl = O.objective(lr.A, lr.E, inst["lam"])
        assert fa == pytest.approx(fl, rel=1e-5), (fa, fl)


def test_adm_converged_multiplier_is_dual_feasible():
    """At the optimum Y is in d||A||_* and in lam d||E||_1: ||Y||_2 <= 1, ||Y||_inf <= lam (E3)."""
    inst = ts.table1_instance(20, 6, 1)
    r, _, _ = _run_adm(inst, rho=1.02, tol=1e-11, max_inner=3000)
    assert r.converged
    assert np.linalg.norm(r.Y, 2) <= 1.0 + 1e-4
    assert np.abs(r.Y).max() <= inst["lam"] * (1.0 + 1e-4)
    # with the default fast penalty (rho = 1.25) feasibility is only approximate
    r2, _, _ = _run_adm(inst)
    assert 1.0 < np.linalg.norm(r2.Y, 2) < 1.1


def test_tilt_with_adm_inner_runs_and_matches_definition():
    """Alg. 1 with the ADM inner loop (the paper's 'ADM' comparison column): cold starts, the
    tau update is the ADM's own dtau; one fixed outer step equals a hand-run ADM at tau0."""
    cfg = ts.CONFIGS[1]
    b = ts.gen_batch(cfg, 0, 1)
    prm = O.Params(inner="adm", fixed_inner_iters=10, fixed_outer_iters=1, max_inner=10, max_outer=1)
    out = O.tilt(b["images"][0], b["boxes"][0], b["tau0"][0], cfg.kind, prm)
    d, jraw, st = O.warp(b["images"][0], b["boxes"][0], b["tau0"][0].astype(np.float64), cfg.kind)
    dh, j, _ = O.normalise(d, jraw)
    proj = O.Projector(j, O.constraints_q(b["tau0"][0].astype(np.float64), cfg.kind, 32, 32))
    mu0 = 1.25 / np.linalg.svd(dh, compute_uv=False)[0]
    r = O.adm(dh, proj, 1 / math.sqrt(32), mu0, 1.25, 1e-6, 10, fixed_iters=10)
    np.testing.assert_allclose(out["A"], r.A, atol=1e-12)
    np.testing.assert_allclose(out["tau"], b["tau0"][0] + r.dtau, atol=1e-12)
