"""End-to-end GPU parity of tilt_solve_batch (the hot entry) against the fp64 oracle.

Protocol:
* fixed count: one outer iteration with exactly K inner iterations and the oracle's rho decisions
  replayed: A and E within 1e-4 relative Frobenius (BASELINE.json north_star);
* convergence: the oracle runs free; the GPU replays its outer-iteration count; tau within 1e-3
  max-abs (normalised coordinates), rank of A equal (outside the Z19 band), objective within 1e-3;
* full size: config 2's 1024-patch batch in the bench launch configuration, sampled patches vs
  the oracle plus properties that hold for every patch;
* edge cases: empty batch, ragged/odd sizes, m != n, failures (escape, zero patch, singular Gram),
  sharding determinism, the 2-level pyramid.
"""
import dataclasses

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
    s = T.TiltSolver(0, max_batch=1024, max_m=128, max_n=128, max_p=8, max_image_elems=64 * 200 * 200)
    yield s
    s.close()


def _replay_tensor(traces_per_patch, max_outer, max_inner, stops=False):
    """Replay bytes (reading Z21): bit 0 = the oracle's rho decision, bit 1 = its inner loop ended."""
    import torch
    B = len(traces_per_patch)
    arr = np.zeros((B, max_outer, max_inner), np.uint8)
    for b, trs in enumerate(traces_per_patch):
        for it, tr in enumerate(trs):
            arr[b, it, :len(tr)] = [t[3] for t in tr]
            if stops and len(tr):
                arr[b, it, len(tr) - 1] |= 2
    return torch.as_tensor(arr, device="cuda")


@pytest.mark.parametrize("path,ns", [(1, 1), (1, 4)])
@pytest.mark.parametrize("cfg_id,K", [(1, 20), (1, 50), (2, 20), (2, 50)])
def test_fixed_count_parity(solver, T, cfg_id, K, path, ns):
    """path 1: CTA-per-patch kernel (tilt_params.kernel_path);
    ns: Newton-Schulz period of the carried V (tilt_params.ns_period)."""
    cfg = ts.CONFIGS[cfg_id]
    B = 4
    b = ts.gen_batch(cfg, 0, B)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1)
    refs = [O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, prm_o) for k in range(B)]
    rr = _replay_tensor([r["traces"] for r in refs], 1, K)
    prm = T.default_params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1, kernel_path=path,
                           ns_period=ns)
    prm.rho_replay = rr.data_ptr()
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm, want_Y=True)
    rep = T.reports_to_numpy(out["rep"])
    assert np.all(rep["kernel_path"] == path)
    for k in range(B):
        a = out["A"][k].double().cpu().numpy()
        e = out["E"][k].double().cpu().numpy()
        ra = np.linalg.norm(a - refs[k]["A"]) / np.linalg.norm(refs[k]["A"])
        re = np.linalg.norm(e - refs[k]["E"]) / np.linalg.norm(refs[k]["E"])
        assert ra < 1e-4 and re < 1e-4, (cfg_id, K, k, ra, re)
        tau = out["tau"][k].double().cpu().numpy()
        assert np.max(np.abs(tau - refs[k]["tau"])) < 1e-3
        assert rep["inner_iters"][k] == K and rep["outer_iters"][k] == 1


def test_fixed_count_parity_own_jacobi_oracle(solver, T):
    """Fixed-count parity against the oracle running its own one-sided Jacobi SVD (Params.svd)."""
    cfg = ts.CONFIGS[1]
    K, B = 20, 2
    b = ts.gen_batch(cfg, 0, B)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1, svd="jacobi")
    refs = [O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, prm_o) for k in range(B)]
    rr = _replay_tensor([r["traces"] for r in refs], 1, K)
    prm = T.default_params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1)
    prm.rho_replay = rr.data_ptr()
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    for k in range(B):
        a = out["A"][k].double().cpu().numpy()
        e = out["E"][k].double().cpu().numpy()
        assert np.linalg.norm(a - refs[k]["A"]) < 1e-4 * np.linalg.norm(refs[k]["A"])
        assert np.linalg.norm(e - refs[k]["E"]) < 1e-4 * np.linalg.norm(refs[k]["E"])


def _convergence_case(solver, T, cfg, idx_list, replay=True, path=0, **gen):
    """Oracle free-running; the GPU replays its outer count and (replay=True) its rho decisions and
    inner-loop ends (parity protocol 3 of SURVEY.md §8(c): the outer problem is flat along the aspect
    direction, so only a replayed path is comparable to 1e-3)."""
    b = ts.gen_batch(cfg, idx_list[0], len(idx_list), **gen)
    refs = [O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind) for k in range(len(idx_list))]
    results = []
    for k, r in enumerate(refs):
        prm = T.default_params(fixed_outer_iters=max(1, r["outer_iters"]), kernel_path=path)
        if replay:
            rr = _replay_tensor([r["traces"]], prm.max_outer, prm.max_inner, stops=True)
            prm.rho_replay = rr.data_ptr()
        out = solver.solve(b["images"][k:k + 1], [0], b["boxes"][k:k + 1], b["tau0"][k:k + 1], cfg.kind, prm)
        rep = T.reports_to_numpy(out["rep"])[0]
        tau = out["tau"][0].double().cpu().numpy()
        results.append((r, rep, tau))
    return results


def _disagreements(res):
    bad = []
    for k, (r, rep, tau) in enumerate(res):
        dt = np.max(np.abs(tau - r["tau"]))
        dobj = abs(rep["objective"] - r["objective"]) / r["objective"]
        rank_ok = (rep["rank"] == r["rank"]) or r["rank_band"] or rep["rank_band"]
        if not (dt < 1e-3 and dobj < 1e-3 and rank_ok):
            bad.append((k, dt, dobj, int(rep["rank"]), r["rank"], r["outer_iters"], r["stop_rule"]))
    return bad


@pytest.mark.parametrize("path", [1])
@pytest.mark.parametrize("cfg_id", [1, 2])
def test_convergence_parity(solver, T, cfg_id, path):
    """tau within 1e-3 max-abs, rank equal, objective within 1e-3 (BASELINE north_star), replayed path."""
    cfg = ts.CONFIGS[cfg_id]
    res = _convergence_case(solver, T, cfg, list(range(8 if cfg_id == 1 else 3)), path=path)
    bad = _disagreements(res)
    for r, rep, _ in res:
        assert rep["inner_iters"] == r["inner_iters"] and rep["outer_iters"] == r["outer_iters"]
    assert not bad, bad


def _unstable(cfg, idx, r, rel=1e-7):
    """Reading Z22: the fp64 oracle's own tau moves by > 1e-3 when its input is perturbed by 1e-7
    relative (same outer count): a basin-edge patch, excluded from tau parity and counted."""
    b = ts.gen_batch(cfg, idx, 1)
    rng = np.random.default_rng([22, idx])
    img = b["images"][0] * (1.0 + rel * rng.standard_normal(b["images"][0].shape))
    prm = O.Params(fixed_outer_iters=max(1, r["outer_iters"]), max_outer=max(1, r["outer_iters"]))
    rp = O.tilt(img, b["boxes"][0], b["tau0"][0], cfg.kind, prm)
    return float(np.max(np.abs(rp["tau"] - r["tau"]))) > 1e-3


def test_convergence_free_running(solver, T):
    """Free-running rho decisions (only the outer count replayed): fp32 vs fp64 branch flips
    (reading Z21) can move the flat aspect direction. Disagreeing patches are classified by Z22;
    the stable ones must agree (at most one fp32 branch-flip case among 8 is tolerated)."""
    cfg = ts.CONFIGS[1]
    res = _convergence_case(solver, T, cfg, list(range(8)), replay=False)
    bad = _disagreements(res)
    unstable = [d for d in bad if _unstable(cfg, d[0], res[d[0]][0])]
    stable_bad = [d for d in bad if d not in unstable]
    print(f"free-running: {len(bad)} of 8 disagree, {len(unstable)} of them unstable (Z22)")
    assert len(bad) <= 3, bad
    assert len(stable_bad) <= 1, (stable_bad, unstable)


def test_full_size_config2(solver, T):
    """Config 2 (1024 x 50x50 homography) in the bench launch configuration."""
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, 0, cfg.batch)
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind)
    rep = T.reports_to_numpy(out["rep"])
    tau = out["tau"].double().cpu().numpy()
    assert np.all(np.isfinite(tau))
    assert set(np.unique(rep["status"])) <= {T.CONVERGED, T.MAX_OUTER, T.WINDOW_ESCAPE}
    conv = rep["status"] == T.CONVERGED
    assert conv.mean() > 0.5
    ok = rep["status"] <= T.MAX_OUTER
    assert np.all(rep["outer_iters"][ok] >= 1) and np.all(rep["inner_iters"][ok] >= rep["outer_iters"][ok])
    assert np.all(np.abs(rep["patch_norm"][ok]) > 0)
    # determinism: the same batch solved again gives identical bits (persistent queue order-free)
    out2 = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind)
    assert np.array_equal(out2["tau"].cpu().numpy(), out["tau"].cpu().numpy())
    assert np.array_equal(out2["A"].cpu().numpy(), out["A"].cpu().numpy())
    # sampled patches vs the oracle (outer count replayed)
    for k in (0, 517):
        r = O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind)
        prm = T.default_params(fixed_outer_iters=max(1, r["outer_iters"]))
        rr = _replay_tensor([r["traces"]], prm.max_outer, prm.max_inner, stops=True)
        prm.rho_replay = rr.data_ptr()
        o1 = solver.solve(b["images"][k:k + 1], [0], b["boxes"][k:k + 1], b["tau0"][k:k + 1], cfg.kind, prm)
        t1 = o1["tau"][0].double().cpu().numpy()
        rep1 = T.reports_to_numpy(o1["rep"])[0]
        assert np.max(np.abs(t1 - r["tau"])) < 1e-3, (k, t1, r["tau"])
        assert abs(rep1["objective"] - r["objective"]) < 1e-3 * r["objective"]
        # the same patch inside the full batch ran free: its status is a valid outcome
        assert rep["status"][k] in (T.CONVERGED, T.MAX_OUTER, T.WINDOW_ESCAPE)


def test_sharding_bit_identical(solver, T):
    cfg = ts.CONFIGS[1]
    b = ts.gen_batch(cfg, 0, 6)
    prm = T.default_params(max_outer=5)
    full = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    for sl in (slice(0, 2), slice(2, 6)):
        part = solver.solve(b["images"], b["patch_image"][sl], b["boxes"][sl], b["tau0"][sl], cfg.kind,
                            T.default_params(max_outer=5))
        assert np.array_equal(part["tau"].cpu().numpy(), full["tau"][sl].cpu().numpy())
        assert np.array_equal(part["E"].cpu().numpy(), full["E"][sl].cpu().numpy())


def test_edge_cases(solver, T):
    import torch
    cfg = ts.CONFIGS[1]
    # empty batch is a no-op
    b = ts.gen_batch(cfg, 0, 3)
    out = solver.solve(b["images"], b["patch_image"][:0], b["boxes"][:0], b["tau0"][:0], cfg.kind,
                       T.default_params(win_h=32, win_w=32))
    assert out["tau"].shape == (0, 6)
    # failure statuses never abort the batch
    imgs = b["images"].copy()
    imgs[1] = 0.0                        # zero patch
    imgs[2] = 0.5                        # constant image: J = 0, Gram singular
    tau0 = b["tau0"].copy()
    tau0[0, 4] = 1.5                     # window escapes the canvas
    out = solver.solve(imgs, b["patch_image"], b["boxes"], tau0, cfg.kind, T.default_params(max_outer=3))
    rep = T.reports_to_numpy(out["rep"])
    assert rep["status"].tolist() == [T.WINDOW_ESCAPE, T.ZERO_PATCH, T.SINGULAR_GRAM]
    np.testing.assert_allclose(out["tau"][0].cpu().numpy(), tau0[0], atol=0)
    # bad arguments
    with pytest.raises(T.TiltError):
        solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind,
                     T.default_params(rho0=0.5))
    del torch


@pytest.mark.parametrize("m,n,kind", [(33, 33, O.AFFINE), (40, 56, O.HOMOGRAPHY), (63, 45, O.AFFINE),
                                      # size-class edges, where dynamic + static shared memory crosses
                                      # the 48 KB default (the 32 x 32 homography once failed there)
                                      (32, 32, O.HOMOGRAPHY), (61, 61, O.HOMOGRAPHY), (62, 60, O.AFFINE),
                                      (64, 64, O.HOMOGRAPHY), (128, 128, O.HOMOGRAPHY)])
def test_ragged_sizes_fixed_count(solver, T, m, n, kind):
    cfg = dataclasses.replace(ts.CONFIGS[1], m=m, n=n, kind=kind, config_id=950 + m)
    B, K = 2, 20
    b = ts.gen_batch(cfg, 0, B)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=2, max_inner=K, max_outer=2)
    refs = [O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], kind, prm_o) for k in range(B)]
    rr = _replay_tensor([r["traces"] for r in refs], 2, K)
    prm = T.default_params(fixed_inner_iters=K, fixed_outer_iters=2, max_inner=K, max_outer=2)
    prm.rho_replay = rr.data_ptr()
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], kind, prm)
    for k in range(B):
        a = out["A"][k].double().cpu().numpy()
        ra = np.linalg.norm(a - refs[k]["A"]) / np.linalg.norm(refs[k]["A"])
        assert ra < 1e-3, (m, n, k, ra)  # two outer iterations: the Y~ warm start carries fp32 noise
        assert np.max(np.abs(out["tau"][k].double().cpu().numpy() - refs[k]["tau"])) < 1e-3


@pytest.mark.parametrize("path", [1, 3])
@pytest.mark.parametrize("warm", [0, 1])
def test_pyramid_config3_small(solver, T, warm, path):
    """2-level pyramid (reading Z18); warm = 1: the fine level starts from the coarse A, E, Y (Z26).
    path 1: CTA-per-patch kernels; path 3: the multi-CTA path (the auto route above 128 x 128),
    which must honour the warm start too."""
    cfg = ts.CONFIGS[3]
    B, K = 2, 20
    b = ts.gen_batch(cfg, 0, B)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=2, max_inner=K, max_outer=2, pyramid_warm=bool(warm))
    refs = [O.tilt_pyramid(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, prm_o, levels=2)
            for k in range(B)]
    prm = T.default_params(fixed_inner_iters=K, fixed_outer_iters=2, max_inner=K, max_outer=2, pyramid_levels=2,
                           pyramid_warm=warm, kernel_path=path)
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    rep = T.reports_to_numpy(out["rep"])
    for k in range(B):
        assert np.max(np.abs(out["tau"][k].double().cpu().numpy() - refs[k]["tau"])) < 1e-3
        a = out["A"][k].double().cpu().numpy()
        assert np.linalg.norm(a - refs[k]["A"]) / np.linalg.norm(refs[k]["A"]) < 1e-3
        assert rep["outer_iters"][k] == 4 and rep["inner_iters"][k] == 4 * K


@pytest.fixture(scope="module")
def solver_big(T):
    s = T.TiltSolver(0, max_batch=4, max_m=200, max_n=200, max_p=8, max_image_elems=4 * 400 * 400)
    yield s
    s.close()


@pytest.mark.parametrize("cfg_id,path", [(3, 1), (4, 1), (4, 3), (4, 0)])
def test_fixed_count_parity_large_configs(solver_big, T, cfg_id, path):
    """Configs 3 (100x100 homography, fine level without the pyramid: the S128 CTA class) and 4
    (200x200 affine): path 1 forces the CTA-per-patch S256 class (B in shared memory, V and S in the
    workspace), path 3 the multi-CTA path, path 0 the auto route (multi-CTA above 128 x 128). One
    outer iteration of 20 LADMAP iterations with replayed rho, A and E within 1e-4 of the oracle."""
    cfg = ts.CONFIGS[cfg_id]
    B, K = 2, 20
    b = ts.gen_batch(cfg, 0, B)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1)
    refs = [O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, prm_o) for k in range(B)]
    rr = _replay_tensor([r["traces"] for r in refs], 1, K)
    prm = T.default_params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1, kernel_path=path)
    prm.rho_replay = rr.data_ptr()
    out = solver_big.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    rep = T.reports_to_numpy(out["rep"])
    assert np.all(rep["kernel_path"] == (path if path else (3 if cfg.m > 128 else 1)))
    for k in range(B):
        a = out["A"][k].double().cpu().numpy()
        e = out["E"][k].double().cpu().numpy()
        ra = np.linalg.norm(a - refs[k]["A"]) / np.linalg.norm(refs[k]["A"])
        re = np.linalg.norm(e - refs[k]["E"]) / np.linalg.norm(refs[k]["E"])
        assert ra < 1e-4 and re < 1e-4, (cfg_id, k, ra, re)
        assert np.max(np.abs(out["tau"][k].double().cpu().numpy() - refs[k]["tau"])) < 1e-3


def test_host_buffer_entry_matches_device_entry(solver, T):
    """tilt_solve_batch_host (the end-to-end entry: host buffers, copies inside) gives the same bits
    as tilt_solve_batch on device buffers (the persistent kernel is deterministic per patch)."""
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, 0, 8)
    prm = T.default_params(fixed_inner_iters=10, fixed_outer_iters=2, max_inner=10, max_outer=2)
    d = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    h = solver.solve_host(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    assert np.array_equal(h["tau"], d["tau"].cpu().numpy())
    assert np.array_equal(h["A"], d["A"].cpu().numpy()) and np.array_equal(h["E"], d["E"].cpu().numpy())
    rep_d = T.reports_to_numpy(d["rep"])
    assert np.array_equal(h["rep"]["inner_iters"], rep_d["inner_iters"])
    assert np.array_equal(h["rep"]["status"], rep_d["status"])


def test_bad_box_and_params_not_mutated(solver, T):
    """Every box of a call must be win_w x win_h: a patch whose box differs gets TILT_PATCH_BAD_BOX
    and is not solved (tau_out = tau0), the others are unaffected; the binding never writes the
    caller's params (a reused object must not carry one call's window size into the next)."""
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, 0, 3)
    prm = T.default_params(max_outer=2, fixed_outer_iters=2, fixed_inner_iters=10, max_inner=10)
    ref = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    assert prm.win_h == 0 and prm.win_w == 0
    boxes = b["boxes"].copy()
    boxes[1, 2] -= 2
    prm.win_h, prm.win_w = cfg.m, cfg.n
    out = solver.solve(b["images"], b["patch_image"], boxes, b["tau0"], cfg.kind, prm)
    rep = T.reports_to_numpy(out["rep"])
    assert list(rep["status"]) == [rep["status"][0], T.BAD_BOX, rep["status"][2]]
    assert rep["status"][0] != T.BAD_BOX
    np.testing.assert_array_equal(out["tau"][1].cpu().numpy(), b["tau0"][1].astype(np.float32))
    for k in (0, 2):
        np.testing.assert_array_equal(out["tau"][k].cpu().numpy(), ref["tau"][k].cpu().numpy())
