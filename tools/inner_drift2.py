"""Drift of the fp32 LADMAP iterate from the fp64 one far into an inner loop, on the inner entry
(tilt_inner_batch: explicit projector from a given J, Q) vs the solve path (implicit projector):
the oracle's D_hat, J, Q of a config-2 patch at tau0, rho replayed, K up to 800."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import tilt_synth as ts  # noqa: E402


def main():
    import paper_1205_5351_b200 as T
    cfg = ts.CONFIGS[2]
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 21
    b = ts.gen_batch(cfg, idx, 1)
    d, jraw, st = O.warp(b["images"][0], b["boxes"][0], b["tau0"][0].astype(np.float64), cfg.kind)
    dh, j, nd = O.normalise(d, jraw)
    q = O.constraints_q(b["tau0"][0].astype(np.float64), cfg.kind, cfg.m, cfg.n)
    dh32, j32, q32 = dh.astype(np.float32), j.astype(np.float32), q.astype(np.float32)
    dh64, j64, q64 = dh32.astype(np.float64), j32.astype(np.float64), q32.astype(np.float64)
    proj = O.Projector(j64, q64)
    s = T.TiltSolver(0, max_batch=4, max_m=64, max_n=64, max_p=8)
    lam = 1 / np.sqrt(50)
    mu0 = 1.25 / np.linalg.svd(dh64, compute_uv=False)[0]
    z = np.zeros_like(dh64)
    for K in (20, 100, 200, 400, 800):
        r = O.ladmap(dh64, proj, lam, mu0, 1e6 * mu0, 2.0, 1e-6, 0.1, K, dh64.copy(), z, z, fixed_iters=K)
        bits = np.array([[t[3] for t in r.trace]], np.uint8)
        prm = T.default_params(fixed_inner_iters=K, max_inner=K)
        out = s.inner(dh32[None], j32[None], Q=q32[None], params=prm, rho_replay=bits)
        a = out["A"][0].double().cpu().numpy()
        e = out["E"][0].double().cpu().numpy()
        print(json.dumps({"K": K, "mu": r.trace[-1][0], "relA": float(np.linalg.norm(a - r.A) / np.linalg.norm(r.A)),
                          "relE": float(np.linalg.norm(e - r.E) / np.linalg.norm(r.E))}), flush=True)


if __name__ == "__main__":
    main()
