"""Pins for the oracle's D o tau, Jacobian and constraint rows.

* identity tau on an integer-aligned window is an exact pixel copy;
* a half-pixel shift of a ramp gives neighbour averages (bilinear closed form);
* J matches central finite differences of the *normalised* warp (Alg. 1 Step 1);
* J is orthogonal to D_hat (quotient rule), ||D_hat|| = 1;
* the Q area row matches finite differences of the shoelace area; affine area gradient is
  proportional to (a22, -a21, -a12, a11, 0, 0) (det of the linear part);
* window escape is reported.
"""
import numpy as np
import pytest

import oracle as O
import tilt_synth as ts


def _smooth_image(hh, ww, seed=0):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:hh, 0:ww].astype(np.float64)
    img = np.zeros((hh, ww))
    for _ in range(4):
        fx, fy, ph = rng.uniform(0.05, 0.3), rng.uniform(0.05, 0.3), rng.uniform(0, 6)
        img += np.sin(fx * x + fy * y + ph)
    return img


@pytest.mark.parametrize("kind", [O.AFFINE, O.HOMOGRAPHY])
def test_identity_is_pixel_copy(kind):
    img = _smooth_image(40, 50)
    box = (7, 5, 20, 16)
    d, jraw, st = O.warp(img, box, ts.identity_tau(kind), kind)
    assert st == O.CONVERGED
    np.testing.assert_array_equal(d, img[5:21, 7:27])
    assert jraw.shape == ((6 if kind == O.AFFINE else 8), 16, 20)


def test_half_pixel_shift_on_ramp():
    img = np.tile(np.arange(30, dtype=np.float64) * 2.0, (20, 1))
    box = (4, 4, 10, 10)
    s = 5.0
    tau = ts.identity_tau(O.AFFINE)
    tau[4] = 0.5 / s  # h13 in normalised units = half a pixel
    d, jraw, st = O.warp(img, box, tau, O.AFFINE)
    np.testing.assert_allclose(d, 0.5 * (img[4:14, 4:14] + img[4:14, 5:15]), atol=1e-12)
    # translation column = s * dI/dX = s * 2 everywhere
    np.testing.assert_allclose(jraw[4], 2.0 * s, atol=1e-12)


@pytest.mark.parametrize("kind", [O.AFFINE, O.HOMOGRAPHY])
def test_jacobian_vs_finite_difference(kind):
    img = _smooth_image(80, 80, seed=3)
    box = (20, 22, 32, 30)
    rng = np.random.default_rng(7)
    tau = ts.identity_tau(kind) + rng.uniform(-0.05, 0.05, size=6 if kind == O.AFFINE else 8)
    if kind == O.HOMOGRAPHY:
        tau[6:] = rng.uniform(-0.02, 0.02, size=2)
    d, jraw, _ = O.warp(img, box, tau, kind)
    dh, j, nd = O.normalise(d, jraw)
    hstep = 1e-6
    for q in range(len(tau)):
        tp, tm = tau.copy(), tau.copy()
        tp[q] += hstep
        tm[q] -= hstep
        dp = O.warp(img, box, tp, kind)[0]
        dm = O.warp(img, box, tm, kind)[0]
        fd_raw = (dp - dm) / (2 * hstep)
        fd = (dp / np.linalg.norm(dp) - dm / np.linalg.norm(dm)) / (2 * hstep)
        # the bilinear interpolant is smooth inside cells; exclude pixels within 1e-4 of a cell edge
        m, n, s, cx, cy, du, dv = O.frame(box)
        h = O.tau_to_h(tau, kind)
        w = 1 + (h[2, 0] * du + h[2, 1] * dv) / s
        xs = cx + (h[0, 0] * du + h[0, 1] * dv + s * h[0, 2]) / w
        ys = cy + (h[1, 0] * du + h[1, 1] * dv + s * h[1, 2]) / w
        ok = (np.abs(xs - np.round(xs)) > 1e-4) & (np.abs(ys - np.round(ys)) > 1e-4)
        assert ok.mean() > 0.95
        np.testing.assert_allclose(jraw[q][ok], fd_raw[ok], rtol=0, atol=1e-6 * np.abs(jraw[q]).max())
        # normalised J vs FD of the normalised warp (pixels near edges perturb the norm by O(h))
        assert np.linalg.norm((j[q] - fd)[ok]) <= 1e-5 * np.linalg.norm(j[q])
    assert np.linalg.norm(dh) == pytest.approx(1.0, abs=1e-14)
    assert np.max(np.abs(np.tensordot(j, dh, axes=([1, 2], [0, 1])))) < 1e-12


def test_constraint_rows():
    rng = np.random.default_rng(9)
    for kind in (O.AFFINE, O.HOMOGRAPHY):
        for m, n in ((32, 32), (40, 56)):
            tau = ts.identity_tau(kind) + rng.uniform(-0.1, 0.1, size=6 if kind == O.AFFINE else 8)
            q = O.constraints_q(tau, kind, m, n)
            np.testing.assert_allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-14)
            assert q[0, 4] == 1.0 and q[1, 5] == 1.0
            fd = np.zeros(len(tau))
            for k in range(len(tau)):
                tp, tm = tau.copy(), tau.copy()
                tp[k] += 1e-6
                tm[k] -= 1e-6
                fd[k] = (O.shoelace_area(tp, kind, m, n) - O.shoelace_area(tm, kind, m, n)) / 2e-6
            np.testing.assert_allclose(q[2], fd / np.linalg.norm(fd), atol=1e-7)
            if kind == O.AFFINE:
                a11, a12, a21, a22 = tau[:4]
                g = np.array([a22, -a21, -a12, a11, 0, 0])
                np.testing.assert_allclose(q[2], g / np.linalg.norm(g), atol=1e-12)


def test_window_escape():
    img = _smooth_image(20, 20)
    tau = ts.identity_tau(O.AFFINE)
    tau[4] = 1.5  # shifts the window by 1.5 s = 7.5 pixels to the right
    _, _, st = O.warp(img, (5, 5, 10, 10), tau, O.AFFINE)
    assert st == O.WINDOW_ESCAPE
    # a window touching the last column escapes (x0 + 1 > W - 1)
    _, _, st = O.warp(img, (10, 5, 10, 10), ts.identity_tau(O.AFFINE), O.AFFINE)
    assert st == O.WINDOW_ESCAPE
