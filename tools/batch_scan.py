"""Per-patch work distribution and batch-size scan of the hot entry (config 2 by default).

Prints, per batch size B: solve time, converged patches/s, inner iterations/s, and the quantiles of
per-patch LADMAP iterations (the tail decides the makespan when B is close to the resident slots).
Usage: python tools/batch_scan.py [--cfg 2] [--sizes 592,1024,2048,4096]
"""
import argparse
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
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--sizes", default="592,1024,2048,4096")
ap.add_argument("--ctas", default="0", help="comma list of tilt_params.ctas_per_sm values")
a = ap.parse_args()
cfg = ts.CONFIGS[a.cfg]
sizes = [int(s) for s in a.sizes.split(",")]
full = bench.gen_shard(a.cfg, 0, max(sizes))
for B, cps in [(B, int(c)) for B in sizes for c in a.ctas.split(",")]:
    b = {k: v[:B] for k, v in full.items()}
    s = T.TiltSolver(0, max_batch=B, max_m=cfg.m, max_n=cfg.n, max_p=cfg.p, max_image_elems=b["images"].size)
    prm = T.default_params(win_h=cfg.m, win_w=cfg.n, ctas_per_sm=cps)
    out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm, sync=False)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    rep = T.reports_to_numpy(out["rep"])
    it = rep["inner_iters"].astype(np.float64)
    conv = int(np.sum(rep["status"] == T.CONVERGED))
    q = np.quantile(it, [0.5, 0.9, 0.99, 1.0])
    print(f"B={B:6d} ctas/SM={cps} t={t:8.3f}s conv/s={conv / t:8.1f} iters/s={it.sum() / t:10.0f} mean_it={it.mean():8.0f} "
          f"p50={q[0]:7.0f} p90={q[1]:7.0f} p99={q[2]:7.0f} max={q[3]:7.0f} "
          f"outer_mean={rep['outer_iters'].mean():5.1f} conv={conv / B:.3f}", flush=True)
    s.close()
