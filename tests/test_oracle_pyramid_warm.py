"""Pins of the pyramid warm start (reading Z26): the fine level's first
inner loop starts from the coarse A, E, Y replicated 2x2 and halved. The paper has no pyramid
(reading Z18), so the pins are the properties the reading is built on: the scaling keeps the norms
that bound the dual, it maps the coarse D_hat exactly onto the fine D_hat of a 2x2-block image, and
the warm start leaves the (convex) first inner problem's optimum unchanged."""
import numpy as np

import oracle as O
import tilt_synth as ts


def test_upsample_keeps_frobenius_and_spectral_norms():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(25, 25))
    u = O.upsample2x_warm(x)
    assert u.shape == (50, 50)
    assert abs(np.linalg.norm(u) / np.linalg.norm(x) - 1) < 1e-14
    assert abs(np.linalg.norm(u, 2) / np.linalg.norm(x, 2) - 1) < 1e-12
    # l_inf halves, so a coarse-feasible dual (|Y| <= lam_c) is fine-feasible (lam_f = lam_c / sqrt 2)
    assert np.max(np.abs(u)) == 0.5 * np.max(np.abs(x))
    # each 2x2 block is constant
    assert np.all(u[0::2, 0::2] == u[1::2, 1::2])


def test_coarse_dhat_maps_onto_fine_dhat_of_a_block_image():
    """Identity tau on a window aligned to 2x2 blocks of a block-constant image: the fine D_hat is
    exactly upsample2x_warm(coarse D_hat) (Alg. 1 Step 1 on both levels, reading Z18's frames)."""
    rng = np.random.default_rng(1)
    coarse = rng.uniform(0.0, 1.0, size=(40, 40))
    fine = np.repeat(np.repeat(coarse, 2, axis=0), 2, axis=1)
    np.testing.assert_array_equal(O.downsample2x(fine), coarse)
    box_f = (20, 16, 32, 36)  # x0, y0 even; w, h even
    box_c = (10, 8, 16, 18)
    tau = np.array([1.0, 0, 0, 1.0, 0, 0])
    d_f, j_f, st_f = O.warp(fine, box_f, tau, O.AFFINE)
    d_c, j_c, st_c = O.warp(coarse, box_c, tau, O.AFFINE)
    assert st_f == O.CONVERGED and st_c == O.CONVERGED
    dh_f, _, _ = O.normalise(d_f, j_f)
    dh_c, _, _ = O.normalise(d_c, j_c)
    np.testing.assert_allclose(dh_f, O.upsample2x_warm(dh_c), atol=1e-15)


def test_warm_start_keeps_the_first_inner_optimum():
    """The first fine inner problem (fixed tau, D_hat, J) is convex: started from the upsampled
    coarse state or cold, LADMAP at tight tolerances reaches the same A, E (P14-style equivalence)."""
    cfg = ts.CONFIGS[3]
    b = ts.gen_batch(cfg, 0, 1)
    img, box, tau0 = b["images"][0], b["boxes"][0], b["tau0"][0]
    prm = O.Params(eps1=1e-9, eps2=1e-4, max_inner=3000, fixed_outer_iters=1, max_outer=1)
    coarse_img = O.downsample2x(img)
    x0, y0, w, h = (int(v) for v in box)
    rc = O.tilt(coarse_img.astype(np.float32).astype(np.float64), (x0 // 2, y0 // 2, w // 2, h // 2), tau0, cfg.kind,
                O.Params(max_outer=3, fixed_outer_iters=3))
    warm = tuple(O.upsample2x_warm(rc[k]) for k in ("A", "E", "Y"))
    cold = O.tilt(img, box, rc["tau"], cfg.kind, prm)
    hot = O.tilt(img, box, rc["tau"], cfg.kind, prm, warm=warm)
    ra = np.linalg.norm(hot["A"] - cold["A"]) / np.linalg.norm(cold["A"])
    re = np.linalg.norm(hot["E"] - cold["E"]) / np.linalg.norm(cold["E"])
    assert ra < 2e-4 and re < 2e-4, (ra, re)
    assert abs(hot["objective"] / cold["objective"] - 1) < 1e-5


def test_pyramid_warm_flag_reaches_the_fine_level():
    cfg = ts.CONFIGS[3]
    b = ts.gen_batch(cfg, 0, 1)
    prm = O.Params(fixed_inner_iters=5, fixed_outer_iters=1, max_inner=5, max_outer=1)
    r0 = O.tilt_pyramid(b["images"][0], b["boxes"][0], b["tau0"][0], cfg.kind, prm, levels=2)
    r1 = O.tilt_pyramid(b["images"][0], b["boxes"][0], b["tau0"][0], cfg.kind,
                        O.Params(**{**prm.__dict__, "pyramid_warm": True}), levels=2)
    np.testing.assert_array_equal(r0["coarse"]["A"], r1["coarse"]["A"])  # same coarse level
    assert np.linalg.norm(r1["A"] - r0["A"]) > 1e-6 * np.linalg.norm(r0["A"])  # different fine start
