"""The seeded input generator (tilt_synth) is deterministic and follows its stated recipe."""
import dataclasses

import numpy as np
import pytest

import tilt_synth as ts


def test_deterministic_per_patch_index():
    cfg = ts.CONFIGS[2]
    a = ts.gen_patch(cfg, 17)
    b = ts.gen_batch(cfg, 15, 4)
    np.testing.assert_array_equal(a["canvas"], b["images"][2])
    np.testing.assert_array_equal(a["tau_g"], b["tau_g"][2])
    assert a["canvas"].dtype == np.float32 and a["canvas"].shape == (100, 100)
    assert tuple(a["box"]) == (25, 25, 50, 50)


def test_corruption_count_exact():
    base = dataclasses.replace(ts.CONFIGS[1], corrupt=0.0, config_id=77)
    corr = dataclasses.replace(base, corrupt=0.25)
    a = ts.gen_patch(base, 3)["canvas"]
    b = ts.gen_patch(corr, 3)["canvas"]
    # the texture is drawn before the corruption, so only the corrupted pixels differ (reading Z23)
    assert np.sum(a != b) <= int(round(0.25 * a.size))
    assert np.sum(a != b) >= int(round(0.25 * a.size)) - 5  # a U[0,1] draw can equal the texel


def test_undeformed_texture_has_rank_r():
    base = dataclasses.replace(ts.CONFIGS[1], corrupt=0.0, config_id=78)
    for r in (2, 3):
        p = ts.gen_patch(base, 0, planted=False, rank=r)
        x0, y0, w, h = p["box"]
        win = p["canvas"][y0:y0 + h, x0:x0 + w].astype(np.float64)
        s = np.linalg.svd(win, compute_uv=False)
        assert np.sum(s > 1e-5 * s[0]) == r


def test_table1_instance_shapes():
    inst = ts.table1_instance(10, 6, 0)
    assert inst["D"].shape == (10, 10) and inst["J"].shape == (6, 10, 10)
    assert np.all(np.abs(inst["D"]) <= 0.5)


def test_recovery_metrics():
    """SURVEY P9(ii) recovery rule and Table 2's error on hand-built transforms:
    tau* = H_G composed with an axis scaling and a translation is recovered (TILT's null
    directions, reading Z10); an extra 3-degree rotation or a perspective error is not."""
    from tilt_synth import metrics as M
    hg = ts.planted_transform(0.3, 0.2, 0.01, -0.02)
    tg = ts.tau_from_h(hg, ts.HOMOGRAPHY)
    assert M.recovered_p9(tg, tg) and M.table2_error(tg, tg) == 0.0
    s = np.diag([1.2, 0.85, 1.0])
    s[0, 2], s[1, 2] = 0.05, -0.03
    assert M.recovered_p9(ts.tau_from_h(hg @ s, ts.HOMOGRAPHY), tg)
    r = ts.planted_transform(np.radians(3.0), 0.0)
    assert not M.recovered_p9(ts.tau_from_h(hg @ r, ts.HOMOGRAPHY), tg)
    p = np.eye(3)
    p[2, 0] = 0.05
    assert not M.recovered_p9(ts.tau_from_h(hg @ p, ts.HOMOGRAPHY), tg)
    t2 = tg.copy()
    t2[0] += 0.1
    assert M.table2_error(t2, tg) == pytest.approx(0.1 / np.linalg.norm(tg))


def test_agree_modulo_aspect():
    """Reading Z10's null direction: an aspect change diag(s, 1/s) is invisible, a skew is not."""
    from tilt_synth import metrics as M
    tg = ts.tau_from_h(ts.planted_transform(0.2, 0.1, 0.01, 0.0), ts.HOMOGRAPHY)
    h = M._h_of(tg) @ np.diag([1.05, 1 / 1.05, 1.0])
    assert M.agree_modulo_aspect(ts.tau_from_h(h, ts.HOMOGRAPHY), tg)
    h2 = M._h_of(tg) @ np.array([[1.0, 0.01, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    assert not M.agree_modulo_aspect(ts.tau_from_h(h2, ts.HOMOGRAPHY), tg)
    h3 = M._h_of(tg) @ np.diag([1.05, 1.0, 1.0])          # not area-preserving
    assert not M.agree_modulo_aspect(ts.tau_from_h(h3, ts.HOMOGRAPHY), tg)
