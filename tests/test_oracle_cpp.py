"""The C++17 oracle twin (oracle/tilt_oracle.cpp, include/tilt_oracle.h) against
the closed forms and against the pinned numpy oracle (oracle/tilt_oracle.py, the same algorithm and
readings). CPU only."""
import numpy as np
import pytest

import oracle as O
import tilt_synth as ts

cpp = pytest.importorskip("oracle.cpp")


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as g
    g.build()


def test_svt_closed_forms_and_lapack():
    a, s, _ = cpp.svt(np.diag([3.0, 1.0]), 2.0)          # P2: diag(3,1), eps 2 -> diag(1,0)
    np.testing.assert_allclose(a, np.diag([1.0, 0.0]), atol=1e-14)
    rng = np.random.default_rng(3)
    for (m, n) in [(7, 5), (5, 7), (40, 40), (30, 12)]:
        M = rng.normal(size=(m, n))
        M[:, -1] = M[:, 0]                                 # rank-deficient
        for eps in (0.0, 0.3, 2.0):
            a, s, _ = cpp.svt(M, eps)
            ref, sref = O.svt(M, eps)
            assert np.linalg.norm(a - ref) <= 1e-12 * max(1.0, np.linalg.norm(ref))
            np.testing.assert_allclose(s, sref[: len(s)], atol=1e-12 * sref[0])


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_fixed_count_matches_numpy_oracle(cfg_id):
    """Two outer iterations of 20 LADMAP iterations (warm starts included): tau, A, E equal to the
    numpy oracle's to rounding."""
    cfg = ts.CONFIGS[cfg_id]
    b = ts.gen_batch(cfg, 0, 2)
    prm = cpp.default_params(fixed_inner=20, max_inner=20, fixed_outer=2, max_outer=2)
    tau, A, E, reps = cpp.solve_batch(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm, n_threads=2)
    po = O.Params(fixed_inner_iters=20, max_inner=20, fixed_outer_iters=2, max_outer=2)
    for k in range(2):
        r = O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind, po)
        np.testing.assert_allclose(tau[k], r["tau"], atol=1e-10)
        assert np.linalg.norm(A[k] - r["A"]) <= 1e-9 * np.linalg.norm(r["A"])
        assert np.linalg.norm(E[k] - r["E"]) <= 1e-9 * np.linalg.norm(r["E"])
        assert reps[k]["outer_iters"] == 2 and reps[k]["inner_iters"] == 40
        assert reps[k]["objective"] == pytest.approx(r["objective"], rel=1e-10)


def test_free_running_matches_numpy_oracle():
    """Algorithm 1 to its stop rule (Z9) on config 1: same outer / inner counts, status, tau."""
    cfg = ts.CONFIGS[1]
    b = ts.gen_batch(cfg, 0, 2)
    tau, A, E, reps = cpp.solve_batch(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, n_threads=2)
    for k in range(2):
        r = O.tilt(b["images"][k], b["boxes"][k], b["tau0"][k], cfg.kind)
        assert reps[k]["status"] == r["status"] and reps[k]["stop_rule"] == r["stop_rule"]
        assert reps[k]["outer_iters"] == r["outer_iters"] and reps[k]["inner_iters"] == r["inner_iters"]
        np.testing.assert_allclose(tau[k], r["tau"], atol=1e-8)
        assert reps[k]["rank"] == r["rank"]


def test_failures_and_arguments():
    cfg = ts.CONFIGS[1]
    b = ts.gen_batch(cfg, 0, 2)
    img = b["images"].astype(np.float64).copy()
    img[1] = 0.0                                          # zero patch
    tau0 = b["tau0"].copy()
    tau0[0, 4] = 5.0                                      # translated far outside: window escape
    prm = cpp.default_params(max_outer=3)
    tau, A, E, reps = cpp.solve_batch(img, b["patch_image"], b["boxes"], tau0, cfg.kind, prm)
    assert reps[0]["status"] == O.WINDOW_ESCAPE and reps[1]["status"] == O.ZERO_PATCH
    boxes = b["boxes"].copy()
    boxes[1, 2] -= 2
    with pytest.raises(ValueError):
        cpp.solve_batch(img, b["patch_image"], boxes, tau0, cfg.kind, prm)
