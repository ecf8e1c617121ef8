"""Step-level GPU parity (through the C ABI) against the fp64 oracle (SURVEY.md §8(c) protocol 1).

K1 warp/Jacobian, K2 projector, the K3 SVT core and the inner loop at a fixed iteration count with
the oracle's rho decisions replayed (reading Z21). Tolerances are derived in DESIGN.md
"Parity tolerances" from fp32 arithmetic (unit roundoff 6e-8) and the iteration counts.
"""
import math

import numpy as np
import pytest

import oracle as O
import tilt_synth as ts

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    import paper_1205_5351_b200 as T
    return T


@pytest.fixture(scope="module")
def solver(T):
    s = T.TiltSolver(0, max_batch=64, max_m=256, max_n=256, max_p=8, max_image_elems=4 * 400 * 400)
    yield s
    s.close()


# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kind", [O.AFFINE, O.HOMOGRAPHY])
def test_warp_jacobian_parity(solver, kind):
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, 0, 6)
    rng = np.random.default_rng(5)
    p = 6 if kind == O.AFFINE else 8
    taus = np.tile(ts.identity_tau(kind), (6, 1))
    taus[1:] += rng.uniform(-0.08, 0.08, size=(5, p))
    if kind == O.HOMOGRAPHY:
        taus[1:, 6:] = rng.uniform(-0.03, 0.03, size=(5, 2))
    taus = taus.astype(np.float32)
    out = solver.warp(b["images"], b["patch_image"], b["boxes"], taus, kind)
    dh = out["Dhat"].double().cpu().numpy()
    J = out["J"].double().cpu().numpy()
    for k in range(6):
        d, jraw, st = O.warp(b["images"][k], b["boxes"][k], taus[k].astype(np.float64), kind)
        assert st == O.CONVERGED and int(out["status"][k]) == O.CONVERGED
        rdh, rj, nd = O.normalise(d, jraw)
        assert abs(float(out["norm"][k]) - nd) <= 1e-6 * nd
        np.testing.assert_allclose(dh[k], rdh, atol=2e-6 * np.abs(rdh).max())
        for q in range(p):
            err = np.linalg.norm(J[k, q] - rj[q]) / np.linalg.norm(rj[q])
            assert err < 1e-5, (k, q, err)


@pytest.mark.parametrize("hw", [(45, 47), (50, 51), (51, 60), (56, 56)])  # 51x60: 48.96 KB of dynamic shared memory, static on top crosses 48 KB
def test_warp_jacobian_parity_ragged_window(solver, hw):
    """K1's scalar store path (m n not a multiple of 4: the 16-byte plane stores need m n % 4 == 0)
    and odd window sizes, homography with perspective terms (the fp32-reciprocal + Newton 1/w), and
    windows whose (d, gx, gy, gz) staging sits at the 48 KB dynamic shared-memory default."""
    cfg = ts.CONFIGS[2]
    kind, p = O.HOMOGRAPHY, 8
    b = ts.gen_batch(cfg, 0, 4)
    m, n = hw
    boxes = b["boxes"].copy()
    boxes[:, 2], boxes[:, 3] = n, m
    rng = np.random.default_rng(11)
    taus = np.tile(ts.identity_tau(kind), (4, 1))
    taus[:, :6] += rng.uniform(-0.05, 0.05, size=(4, 6))
    taus[:, 6:] = rng.uniform(-0.03, 0.03, size=(4, 2))
    taus = taus.astype(np.float32)
    out = solver.warp(b["images"], b["patch_image"], boxes, taus, kind)
    dh = out["Dhat"].double().cpu().numpy().reshape(4, m, n)
    J = out["J"].double().cpu().numpy().reshape(4, p, m, n)
    for k in range(4):
        d, jraw, st = O.warp(b["images"][k], boxes[k], taus[k].astype(np.float64), kind)
        assert st == O.CONVERGED and int(out["status"][k]) == O.CONVERGED
        rdh, rj, nd = O.normalise(d, jraw)
        assert abs(float(out["norm"][k]) - nd) <= 1e-6 * nd
        np.testing.assert_allclose(dh[k], rdh, atol=2e-6 * np.abs(rdh).max())
        for q in range(p):
            assert np.linalg.norm(J[k, q] - rj[q]) < 1e-5 * np.linalg.norm(rj[q]), (k, q)


def test_warp_full_batch_sampled(T):
    """K1 at the bench's full size and launch configuration (config 2: 1024 patches at tau0, the
    roofline_k1 call of bench.py), sampled patches against the oracle's warp."""
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, 0, cfg.batch)
    s = T.TiltSolver(0, max_batch=cfg.batch, max_m=50, max_n=50, max_p=8, max_image_elems=int(b["images"].size))
    out = s.warp(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind)
    dh = out["Dhat"].double().cpu().numpy()
    J = out["J"].double().cpu().numpy()
    assert np.all(out["status"].cpu().numpy() == O.CONVERGED)
    for k in (0, 511, 1023):
        d, jraw, st = O.warp(b["images"][k], b["boxes"][k], b["tau0"][k].astype(np.float64), cfg.kind)
        rdh, rj, nd = O.normalise(d, jraw)
        np.testing.assert_allclose(dh[k], rdh, atol=2e-6 * np.abs(rdh).max())
        for q in range(cfg.p):
            assert np.linalg.norm(J[k, q] - rj[q]) < 1e-5 * np.linalg.norm(rj[q]), (k, q)
    s.close()


def test_warp_escape_and_zero(solver):
    cfg = ts.CONFIGS[1]
    b = ts.gen_batch(cfg, 0, 2)
    imgs = b["images"].copy()
    imgs[1] = 0.0
    taus = np.tile(ts.identity_tau(cfg.kind), (2, 1)).astype(np.float32)
    taus[0, 4] = 1.5  # pushes the window out of the 64x64 canvas
    out = solver.warp(imgs, b["patch_image"], b["boxes"], taus, cfg.kind)
    assert out["status"].cpu().tolist() == [O.WINDOW_ESCAPE, O.ZERO_PATCH]


# ---------------------------------------------------------------------------------------------
SVT_SIZES = [(32, 32), (50, 50), (40, 56), (56, 40), (63, 63), (64, 50), (33, 35), (100, 100), (200, 200)]


@pytest.mark.parametrize("m,n,path", [(m, n, 1) for (m, n) in SVT_SIZES])
def test_svt_parity(solver, m, n, path):
    """path 1: CTA-per-patch kernel (the multi-CTA path's SVT parity is in test_gpu_large.py)."""
    B = 4
    Ms = np.stack([ts.lowrank_sparse(m, n, 3 + k, k) for k in range(B)])
    sig1 = np.array([np.linalg.svd(x, compute_uv=False)[0] for x in Ms])
    eps = (sig1 * np.array([0.01, 0.05, 0.2, 1e-4])).astype(np.float32)
    out = solver.svt(Ms.astype(np.float32), eps, path=path)
    A = out["A"].double().cpu().numpy()
    for k in range(B):
        ref, s = O.svt(Ms[k].astype(np.float32).astype(np.float64), float(eps[k]))
        err = np.linalg.norm(A[k] - ref) / np.linalg.norm(Ms[k])
        assert err < 3e-5, (m, n, k, err)
        gs = np.sort(out["sigma"][k].double().cpu().numpy())[::-1][:min(m, n)]
        np.testing.assert_allclose(gs, s[:min(m, n)], atol=1e-5 * s[0])
    assert int(out["sweeps"].max()) < 20


def test_svt_warm_start_fewer_sweeps(solver):
    m = n = 50
    M0 = ts.lowrank_sparse(m, n, 4, 0)
    rng = np.random.default_rng(0)
    M1 = M0 + 1e-3 * rng.normal(size=(m, n))
    cold = solver.svt(M0[None].astype(np.float32), [1e-3])
    warm = solver.svt(M1[None].astype(np.float32), [1e-3], V=cold["V"])
    ref, _ = O.svt(M1.astype(np.float32).astype(np.float64), 1e-3)
    assert np.linalg.norm(warm["A"][0].double().cpu().numpy() - ref) < 3e-5 * np.linalg.norm(M1)
    assert int(warm["sweeps"][0]) < int(cold["sweeps"][0])


# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("with_q", [False, True])
def test_projector_parity(solver, with_q):
    rng = np.random.default_rng(11)
    B, p, m, n = 3, 8, 50, 50
    J = rng.normal(size=(B, p, m, n))
    v = rng.normal(size=(B, m, n))
    Q = rng.normal(size=(B, 3, p)) if with_q else None
    out = solver.project(J.astype(np.float32), v.astype(np.float32), None if Q is None else Q.astype(np.float32))
    Pv = out["Pv"].double().cpu().numpy()
    dt = out["dtau"].double().cpu().numpy()
    for k in range(B):
        proj = O.Projector(J[k].astype(np.float32).astype(np.float64),
                           None if Q is None else Q[k].astype(np.float32).astype(np.float64))
        vv = v[k].astype(np.float32).astype(np.float64)
        ref = proj.apply(vv)
        assert np.linalg.norm(Pv[k] - ref) <= 1e-5 * np.linalg.norm(vv)
        rdt = proj.delta_tau(vv)
        assert np.linalg.norm(dt[k] - rdt) <= 1e-5 * max(1.0, np.linalg.norm(rdt))


# ---------------------------------------------------------------------------------------------
def _inner_ref(D, J, Q, lam, K, max_inner):
    proj = O.Projector(J, Q)
    sigma1 = np.linalg.svd(D, compute_uv=False)[0]
    mu0 = 1.25 / sigma1
    z = np.zeros_like(D)
    return O.ladmap(D, proj, lam, mu0, 1e6 * mu0, 2.0, 1e-6, 0.1, max_inner, D.copy(), z, z, fixed_iters=K)


@pytest.mark.parametrize("n,p,K", [(10, 6, 20), (50, 6, 20), (50, 6, 50), (32, 8, 50), (100, 6, 20)])
def test_inner_fixed_count_parity_table1_data(solver, T, n, p, K):
    B = 3
    insts = [ts.table1_instance(n, p, s) for s in range(B)]
    D = np.stack([i["D"] for i in insts]).astype(np.float32)
    J = np.stack([i["J"] for i in insts]).astype(np.float32)
    lam = insts[0]["lam"]
    refs = [_inner_ref(D[k].astype(np.float64), J[k].astype(np.float64), None, lam, K, K) for k in range(B)]
    bits = np.array([[t[3] for t in r.trace] for r in refs], np.uint8)
    prm = T.default_params(fixed_inner_iters=K, max_inner=K)
    out = solver.inner(D, J, params=prm, rho_replay=bits, trace=True)
    for k in range(B):
        a = out["A"][k].double().cpu().numpy()
        e = out["E"][k].double().cpu().numpy()
        ra = np.linalg.norm(a - refs[k].A) / np.linalg.norm(refs[k].A)
        re = np.linalg.norm(e - refs[k].E) / max(np.linalg.norm(refs[k].E), 1e-30)
        assert ra < 1e-4 and re < 1e-4, (n, p, K, k, ra, re)
        assert out["rep"]["inner_iters"][k] == K


def test_inner_free_running_table1(solver, T):
    """Statistical pin on the GPU too: objective within 2% of Table 1 at 50x50."""
    B = 10
    insts = [ts.table1_instance(50, 6, s) for s in range(B)]
    D = np.stack([i["D"] for i in insts]).astype(np.float32)
    J = np.stack([i["J"] for i in insts]).astype(np.float32)
    out = solver.inner(D, J)
    rep = out["rep"]
    assert np.all(rep["status"] == T.CONVERGED)
    assert np.mean(rep["objective"]) == pytest.approx(76.6468, rel=0.02)
    assert 12 <= np.mean(rep["inner_iters"]) <= 40
    for k in range(3):  # and the same stop iteration count as the oracle (rho branches agree here)
        r = _inner_ref(D[k].astype(np.float64), J[k].astype(np.float64), None, 1 / math.sqrt(50), 0, 1000)
        assert abs(int(rep["inner_iters"][k]) - r.iters) <= 1
        assert rep["objective"][k] == pytest.approx(O.objective(r.A, r.E, 1 / math.sqrt(50)), rel=1e-4)
