"""Pins for the oracle's outer loop, Algorithm 1.

The outer problem is nonconvex with no closed-form target, so it is pinned by what
the method must do on planted data:
(i)  an undeformed rank-r texture at tau0 = I stays rectified: off-diagonal, translation (and
     perspective) entries stay ~0, the area (centre + area constraints) is preserved
     and the relative rank (reading Z19) equals r. The diagonal (aspect) direction is a null
     direction of the model (reading Z10) and may drift.
(ii) a planted affine / homography deformation A(theta, t) = R(theta)[[1, t], [0, 1]]
      of a clean smooth low-rank texture is recovered up to translation and axis
     scaling (H_G^{-1} tau* diagonal) on most seeds.
(iii) the inner exits satisfy the constraint-residual criterion (Cond1).
"""
import dataclasses

import numpy as np

import oracle as O
import tilt_synth as ts


def _undeformed_cases():
    base = dataclasses.replace(ts.CONFIGS[1], corrupt=0.0, config_id=901)
    for blur in (0.0, 1.0):
        for idx in range(4):
            yield base, idx, blur, 2 + idx % 2


def test_undeformed_texture_stays_rectified():
    for cfg, idx, blur, r in _undeformed_cases():
        p = ts.gen_patch(cfg, idx, planted=False, blur_px=blur, rank=r)
        res = O.tilt(p["canvas"], p["box"], p["tau0"], O.AFFINE)
        tau = res["tau"]
        assert res["status"] == O.CONVERGED
        assert abs(tau[1]) < 1e-4 and abs(tau[2]) < 1e-4          # off-diagonal
        assert abs(tau[4]) < 1e-4 and abs(tau[5]) < 1e-4          # translation (centre row of Q)
        assert abs(tau[0] * tau[3] - tau[1] * tau[2] - 1.0) < 2e-3  # area row of Q
        assert res["rank"] == r and not res["rank_band"]
        assert res["crit1"] < 1e-6                                  # Cond1 at the inner exit


def _recovered(tau, tau_g, kind, off_tol=0.02, persp_tol=1e-2):
    h = np.linalg.inv(O.tau_to_h(tau_g, kind)) @ O.tau_to_h(tau, kind)
    h = h / h[2, 2]
    lin = h[:2, :2]
    off = max(abs(lin[0, 1]) / abs(lin[0, 0]), abs(lin[1, 0]) / abs(lin[1, 1]))
    return off < off_tol and max(abs(h[2, 0]), abs(h[2, 1])) < persp_tol


def test_planted_affine_recovery():
    cfg = dataclasses.replace(ts.CONFIGS[1], corrupt=0.0, config_id=902, rank_lo=2, rank_hi=3)
    ok = 0
    for idx in range(8):
        p = ts.gen_patch(cfg, idx, blur_px=1.0)
        res = O.tilt(p["canvas"], p["box"], p["tau0"], O.AFFINE)
        assert res["status"] in (O.CONVERGED, O.MAX_OUTER)
        ok += _recovered(res["tau"], p["tau_g"], O.AFFINE)
    assert ok >= 6


def test_planted_homography_recovery():
    cfg = dataclasses.replace(ts.CONFIGS[1], corrupt=0.0, config_id=903, rank_lo=2, rank_hi=3,
                              kind=O.HOMOGRAPHY, persp_px=1e-3)
    ok = 0
    for idx in range(8):
        p = ts.gen_patch(cfg, idx, blur_px=1.0)
        res = O.tilt(p["canvas"], p["box"], p["tau0"], O.HOMOGRAPHY)
        assert res["status"] in (O.CONVERGED, O.MAX_OUTER)
        ok += _recovered(res["tau"], p["tau_g"], O.HOMOGRAPHY)
    assert ok >= 6


def test_fixed_counts_and_replay_are_honoured():
    cfg = ts.CONFIGS[1]
    p = ts.gen_patch(cfg, 0)
    prm = O.Params(fixed_inner_iters=7, fixed_outer_iters=3)
    res = O.tilt(p["canvas"], p["box"], p["tau0"], cfg.kind, prm)
    assert res["outer_iters"] == 3 and res["inner_iters"] == 21
    assert all(len(t) == 7 for t in res["traces"])
    # replaying the recorded rho decisions reproduces the run exactly
    bits = [[t[3] for t in tr] for tr in res["traces"]]
    res2 = O.tilt(p["canvas"], p["box"], p["tau0"], cfg.kind, prm, rho_replay=bits)
    np.testing.assert_array_equal(res2["tau"], res["tau"])


def test_pyramid_transfers_tau():
    """Reading Z18: the 2x2-downsampled image at box/2 sees the same normalised frame."""
    cfg = dataclasses.replace(ts.CONFIGS[1], m=64, n=64, corrupt=0.0, config_id=904)
    p = ts.gen_patch(cfg, 0, blur_px=1.0)
    coarse = O.downsample2x(p["canvas"])
    box = p["box"]
    cbox = (box[0] // 2, box[1] // 2, box[2] // 2, box[3] // 2)
    tau = p["tau_g"]
    df, _, _ = O.warp(p["canvas"], box, tau, O.AFFINE)
    dc, _, _ = O.warp(coarse, cbox, tau, O.AFFINE)
    df2 = O.downsample2x(df)
    corr = np.corrcoef(df2.reshape(-1), dc.reshape(-1))[0, 1]
    assert corr > 0.995


def test_oracle_twin_matches_per_patch_tilt():
    """tilt_oracle_solve_batch (SURVEY.md §8(b) oracle twin) = tilt() per patch, incl. the no-state case."""
    cfg = ts.CONFIGS[1]
    b = ts.gen_batch(cfg, 0, 2)
    prm = O.Params(fixed_inner_iters=5, fixed_outer_iters=1, max_inner=5, max_outer=1)
    nimg, H, W = b["images"].shape
    boxes = b["boxes"].copy()
    boxes[1, 0] = W - 5  # the second window leaves the image: WINDOW_ESCAPE, zero A and E
    tau, A, E, reps = O.tilt_oracle_solve_batch(b["images"], nimg, H, W, b["patch_image"], boxes, b["tau0"], 2,
                                                cfg.kind, prm, n_threads=1)
    r0 = O.tilt(b["images"][b["patch_image"][0]], boxes[0], b["tau0"][0], cfg.kind, prm)
    np.testing.assert_array_equal(tau[0], r0["tau"])
    np.testing.assert_array_equal(A[0], r0["A"])
    assert reps[0]["inner_iters"] == 5
    assert reps[1]["status"] == O.WINDOW_ESCAPE and not A[1].any() and not E[1].any()
