"""Parity protocols 2 and 3 of SURVEY.md §8(c) beyond the first inner loop, and sampled parity of
the full-size launches (configs 3 and 5).

* Re-sync (protocol 2): every outer step the oracle starts from the GPU's exported state
  (tau, A, E, Y~) and runs that one step -- the warm start A_0 = A, E_0 = E, Y~_0 = W^TW Y~
   with the new D_hat, J -- with the same fixed inner count; the GPU's own next
  step must agree with it to the fixed-count bar (A, E within 1e-4 relative Frobenius), for 10 outer
  steps. The SVD's carried V is not part of the state the oracle needs: its SVT is the exact
  singular value shrinkage, which is single-valued whatever V seeds the GPU's Jacobi (Z13).
* Full-size launches: the bench's launch configuration (config 5: 65 536 problems; config 3: the
  4096-patch pyramid) with a fixed count, sampled patches vs the oracle.
"""
import multiprocessing as mp
import os

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
    s = T.TiltSolver(0, max_batch=65536, max_m=128, max_n=128, max_p=8, max_image_elems=4096 * 200 * 200)
    yield s
    s.close()


def _gen_one(args):
    cfg_id, idx = args
    return ts.gen_patch(ts.CONFIGS[cfg_id], idx)


def _gen_pool(cfg_id, count):
    """ts.gen_batch(cfg, 0, count) on the host cores (the same patches, generated in parallel)."""
    procs = max(1, min(os.cpu_count() or 1, 32))
    with mp.get_context("fork").Pool(procs) as pool:
        pats = pool.map(_gen_one, [(cfg_id, k) for k in range(count)], chunksize=16)
    return {"images": np.stack([p["canvas"] for p in pats]), "patch_image": np.arange(count, dtype=np.int32),
            "boxes": np.stack([p["box"] for p in pats]), "tau0": np.stack([p["tau0"] for p in pats])}


def _rel(x, ref):
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30))


@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_resync_fixed_count_ten_outer_steps(solver, T, cfg_id):
    """Protocol 2 (re-sync) for 10 outer steps of K = 20 inner iterations, configs 1, 2 and the
    fine level of 3 (100x100, no pyramid); the oracle's rho decisions of each re-synced step are
    replayed on the GPU (Z21)."""
    import torch
    cfg = ts.CONFIGS[cfg_id]
    B, K, S = 2, 20, 10
    b = ts.gen_batch(cfg, 0, B)
    replay = np.zeros((B, S, K), np.uint8)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1)
    tau = [b["tau0"][k].astype(np.float64) for k in range(B)]
    state = [None] * B
    worst = 0.0
    for s in range(S):
        refs = []
        for k in range(B):
            r = O.tilt(b["images"][k], b["boxes"][k], tau[k], cfg.kind, prm_o, warm=state[k])
            assert r["status"] in (O.CONVERGED, O.MAX_OUTER), (cfg_id, s, k, r["status"])
            replay[k, s, :] = [t[3] for t in r["traces"][0]]
            refs.append(r)
        prm = T.default_params(fixed_inner_iters=K, max_inner=K, fixed_outer_iters=s + 1, max_outer=S,
                               pyramid_levels=1)
        rr = torch.as_tensor(replay, device="cuda")
        prm.rho_replay = rr.data_ptr()
        out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm, want_Y=True)
        for k in range(B):
            a = out["A"][k].double().cpu().numpy()
            e = out["E"][k].double().cpu().numpy()
            ra, re = _rel(a, refs[k]["A"]), _rel(e, refs[k]["E"])
            worst = max(worst, ra, re)
            assert ra < 1e-4 and re < 1e-4, (cfg_id, s, k, ra, re)
            t_gpu = out["tau"][k].double().cpu().numpy()
            assert np.max(np.abs(t_gpu - refs[k]["tau"])) < 1e-4, (cfg_id, s, k)
            # re-sync: the next oracle step starts from the GPU's state
            tau[k] = t_gpu
            state[k] = (a, e, out["Y"][k].double().cpu().numpy())
    print(f"config {cfg_id}: re-synced A/E worst relative error over {S} outer steps: {worst:.2e}")


def test_full_batch_config5_launch_sampled(solver, T):
    """65 536 problems in one launch (config 5's batch; 2048 distinct canvases, patch k shows
    canvas k mod 2048): one outer iteration of K = 10 with replayed rho on the sampled patches; A and E
    of the sampled patches within 1e-4 of the oracle, and every copy of a canvas bit-identical
    wherever the persistent queue placed it."""
    import torch
    cfg = ts.CONFIGS[5]
    G, U, K = 65536, 2048, 10
    b = ts.gen_batch(cfg, 0, U)
    pimg = (np.arange(G) % U).astype(np.int32)
    boxes = np.repeat(b["boxes"][:1], G, axis=0)
    tau0 = np.repeat(b["tau0"][:1], G, axis=0)
    samples = [0, 777, 2047]
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1)
    refs = {k: O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, prm_o) for k in samples}
    replay = np.zeros((G, 1, K), np.uint8)
    for k, r in refs.items():
        replay[k::U, 0, :] = [t[3] for t in r["traces"][0]]
    rr = torch.as_tensor(replay, device="cuda")
    prm = T.default_params(fixed_inner_iters=K, max_inner=K, fixed_outer_iters=1, max_outer=1)
    prm.rho_replay = rr.data_ptr()
    out = solver.solve(b["images"], pimg, boxes, tau0, cfg.kind, prm)
    rep = T.reports_to_numpy(out["rep"])
    assert np.all(rep["outer_iters"] == 1) and np.all(rep["inner_iters"] == K)
    for k, r in refs.items():
        for c in (k, k + U, k + 31 * U):
            a = out["A"][c].double().cpu().numpy()
            e = out["E"][c].double().cpu().numpy()
            assert _rel(a, r["A"]) < 1e-4 and _rel(e, r["E"]) < 1e-4, (k, c)
    A = out["A"].view(G // U, U, -1)
    assert bool(torch.all(A == A[0:1]).item())  # every copy bit-identical (rho replay equal per canvas)


def test_full_batch_config3_pyramid_sampled(solver, T):
    """Config 3's full batch (4096 x 100x100 homography, 2-level pyramid) in one call with a fixed
    count (1 outer iteration of K = 10 per level); sampled patches vs oracle.tilt_pyramid: tau within
    1e-3 and A within 1e-3 (two chained levels; the coarse level's rho runs free, Z21)."""
    cfg = ts.CONFIGS[3]
    K = 10
    b = _gen_pool(3, cfg.batch)
    prm = T.default_params(fixed_inner_iters=K, max_inner=K, fixed_outer_iters=1, max_outer=1, pyramid_levels=2)
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    rep = T.reports_to_numpy(out["rep"])
    ok = rep["status"] <= T.MAX_OUTER
    assert ok.mean() > 0.9
    assert np.all(rep["outer_iters"][ok] == 2) and np.all(rep["inner_iters"][ok] == 2 * K)
    prm_o = O.Params(fixed_inner_iters=K, fixed_outer_iters=1, max_inner=K, max_outer=1)
    for k in (0, 1234, 4095):
        if not ok[k]:
            continue
        r = O.tilt_pyramid(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, prm_o, levels=2)
        assert np.max(np.abs(out["tau"][k].double().cpu().numpy() - r["tau"])) < 1e-3, k
        assert _rel(out["A"][k].double().cpu().numpy(), r["A"]) < 1e-3, k


# ------------------------------------------------------------------------------------------------
# Protocol 3, free-running: 64 config-2 patches
# ------------------------------------------------------------------------------------------------
def _oracle_run(args):
    """oracle.tilt on patch idx of config 2: free (replay None) or replaying a GPU run's discrete
    decisions (its outer count, per-outer inner-loop lengths and rho bits)."""
    idx, replay, noise_seed = args
    cfg = ts.CONFIGS[2]
    p = ts.gen_patch(cfg, idx)
    from threadpoolctl import threadpool_limits
    try:
        with threadpool_limits(1):  # one BLAS thread per worker process
            if replay is None:
                r = O.tilt(p["canvas"], p["box"], p["tau0"], cfg.kind)
            else:
                n_outer, counts, bits = replay
                prm = O.Params(fixed_outer_iters=n_outer, max_outer=n_outer, tau_noise=1e-5 if noise_seed else 0.0,
                               noise_seed=noise_seed)
                r = O.tilt(p["canvas"], p["box"], p["tau0"], cfg.kind, prm, rho_replay=bits, inner_replay=counts)
    except Exception as exc:  # reported with the patch index by the test
        raise RuntimeError(f"oracle failed on patch {idx} (replay={replay is not None}): {exc!r}") from None
    return {k: r[k] for k in ("tau", "objective", "rank", "rank_band", "outer_iters", "inner_iters", "status")}


def _agree(rep, tau, r):
    dt = float(np.max(np.abs(tau - r["tau"])))
    dobj = abs(float(rep["objective"]) - r["objective"]) / r["objective"]
    rank_ok = (rep["rank"] == r["rank"]) or r["rank_band"] or rep["rank_band"]
    return dt < 1e-3 and dobj < 1e-3 and rank_ok, dt, dobj


def _agree_modulo_aspect(rep, tau, r):
    """tau equal up to the aspect null direction (Z10), objective 1e-3, rank equal."""
    from tilt_synth.metrics import agree_modulo_aspect
    dobj = abs(float(rep["objective"]) - r["objective"]) / r["objective"]
    rank_ok = (rep["rank"] == r["rank"]) or r["rank_band"] or rep["rank_band"]
    return agree_modulo_aspect(tau, r["tau"]) and dobj < 1e-3 and rank_ok


def test_free_running_convergence_config2_64(solver, T):
    """Protocol 3 on 64 config-2 patches, the GPU free-running with the bench's parameters (its own
    rho decisions, inner-loop ends and outer stop). Checked: the oracle replaying the GPU's
    discrete decisions (outer count, every inner loop's length, every rho bit; readings Z9, Z21)
    reaches the same tau (1e-3 max-abs; for at least 85% of the patches exactly, for the others up
    to the aspect null direction of reading Z10), objective (1e-3) and rank (outside the Z19 band)
    on every patch that is not chain-sensitive -- the GPU computes the paper's method along its own
    decision path. Chain-sensitive (reading Z22): the oracle's own replayed tau moves by > 1e-3 when tau is
    perturbed by 1e-5 relative after every outer step (the size of the fp32-vs-fp64 per-step
    difference: re-synced A, E agree to ~1.4e-5 after 20 inner iterations, test above, and to ~1e-4
    deep in an inner loop at mu ~1e6, tools/inner_drift.py); such patches are counted. Printed: the
    agreement with the oracle's own free-running decisions (the fp32 Cond1/Cond2 statistics decide
    some inner loops differently from fp64, and the outer dynamics carry the difference along the
    flat aspect direction, SURVEY.md §8(c) protocol 3 hazard)."""
    import torch
    cfg = ts.CONFIGS[2]
    N = 64
    b = ts.gen_batch(cfg, 0, N)
    prm = T.default_params()
    trace = torch.full((N, prm.max_outer, prm.max_inner, 4), float("nan"), device="cuda")
    prm.trace = trace.data_ptr()
    out = solver.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    reps = T.reports_to_numpy(out["rep"])
    taus = out["tau"].double().cpu().numpy()
    tr = trace.cpu().numpy()
    jobs = []
    ks = [k for k in range(N) if reps["status"][k] in (T.CONVERGED, T.MAX_OUTER)]
    for k in ks:
        n_outer = int(reps["outer_iters"][k])
        counts = [int(np.sum(np.isfinite(tr[k, i, :, 0]))) for i in range(n_outer)]
        bits = [[int(x) & 1 for x in tr[k, i, :counts[i], 3]] for i in range(n_outer)]
        jobs.append((k, (n_outer, counts, bits), 0))
    procs = max(1, min(os.cpu_count() or 1, 32))
    with mp.get_context("fork").Pool(procs) as pool:
        replayed = pool.map(_oracle_run, jobs, chunksize=1)
        free = pool.map(_oracle_run, [(k, None, 0) for k in ks], chunksize=1)
        bad_replayed, bad_free = [], []
        for j, k in enumerate(ks):
            ok, dt, dobj = _agree(reps[k], taus[k], replayed[j])
            if not ok:
                bad_replayed.append((j, k, dt, dobj, int(reps["rank"][k]), replayed[j]["rank"]))
        noisy = pool.map(_oracle_run, [(jobs[j][0], jobs[j][1], seed) for j, *_ in bad_replayed for seed in (1, 2)],
                         chunksize=1)
    sensitive = []
    for q, (j, k, *_) in enumerate(bad_replayed):
        moves = [float(np.max(np.abs(noisy[2 * q + t]["tau"] - replayed[j]["tau"]))) for t in (0, 1)]
        if max(moves) > 1e-3:
            sensitive.append(k)
    aspect_only = [d[1] for d in bad_replayed if d[1] not in sensitive and
                   _agree_modulo_aspect(reps[d[1]], taus[d[1]], replayed[d[0]])]
    stable_bad = [d[1:] for d in bad_replayed if d[1] not in sensitive and d[1] not in aspect_only]
    for j, k in enumerate(ks):
        ok, dt, dobj = _agree(reps[k], taus[k], free[j])
        if not ok:
            bad_free.append((k, round(dt, 5), int(reps["inner_iters"][k]), free[j]["inner_iters"]))
    caps = int(np.sum(np.sum(np.isfinite(tr[ks, :, :, 0]), axis=2) == prm.max_inner))
    print(f"free-running config 2, {len(ks)} patches: GPU vs oracle replaying the GPU's decisions: "
          f"{len(ks) - len(bad_replayed)} agree, {len(sensitive)} chain-sensitive (Z22) excluded {sensitive}, "
          f"{len(aspect_only)} agree up to the aspect null direction (Z10) {aspect_only}; "
          f"GPU vs the oracle's own decisions: {len(ks) - len(bad_free)} agree (disagreeing: {bad_free}); "
          f"GPU inner loops ending at max_inner: {caps}")
    assert len(ks) - len(bad_replayed) >= 0.85 * len(ks)
    assert not stable_bad, stable_bad
