"""Free-running config-5 patches at several Jacobi tolerances (reading Z14's default vs looser):
time, converged fraction, inner iterations, sweeps per SVT, and the tau change vs the default.
Usage: python tools/jtol_probe.py [--batch 4096] [--tols 0,1e-5,3e-5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--tols", default="0,1e-5,3e-5")
a = ap.parse_args()
cfg = ts.CONFIGS[5]
B = a.batch
b = bench.gen_shard(5, range(B))
s = T.TiltSolver(0, max_batch=B, max_m=cfg.m, max_n=cfg.n, max_p=cfg.p, max_image_elems=int(b["images"].size))
args = [torch.as_tensor(b["images"], device="cuda"), torch.arange(B, dtype=torch.int32, device="cuda"),
        torch.as_tensor(b["boxes"], device="cuda"), torch.as_tensor(b["tau0"], device="cuda")]
ref = None
for tol in [float(t) for t in a.tols.split(",")]:
    prm = T.default_params(win_h=cfg.m, win_w=cfg.n, jacobi_tol=tol)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(*args, cfg.kind, prm, sync=False)
    e1.record()
    torch.cuda.synchronize()
    rep = T.reports_to_numpy(out["rep"])
    tau = out["tau"].double().cpu().numpy()
    if ref is None:
        ref = tau
    it = rep["inner_iters"].sum()
    print(json.dumps({"jacobi_tol": tol, "seconds": e0.elapsed_time(e1) / 1e3,
                      "converged": int((rep["status"] == T.CONVERGED).sum()),
                      "mean_inner": float(it / B), "sweeps_per_svt": float(rep["jacobi_sweeps"].sum() / it),
                      "tau_maxdiff_vs_first": float(np.abs(tau - ref).max()),
                      "tau_frac_within_1e-3": float(np.mean(np.abs(tau - ref).max(axis=1) <= 1e-3))}), flush=True)
