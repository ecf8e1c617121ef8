"""Short, deterministic launch of the hot kernel for ncu (fixed counts so a launch takes ~ms).

Usage: python tools/prof_solve.py [--batch 296] [--inner 30] [--outer 1] [--cfg 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=296)
ap.add_argument("--inner", type=int, default=30)
ap.add_argument("--outer", type=int, default=1)
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--path", type=int, default=0, help="tilt_params.kernel_path (0 auto, 1 CTA, 2 warp)")
ap.add_argument("--ns", type=int, default=1, help="tilt_params.ns_period")
ap.add_argument("--max-sweeps", type=int, default=0, help="tilt_params.jacobi_max_sweeps (0: default)")
ap.add_argument("--jtol", type=float, default=0.0, help="tilt_params.jacobi_tol (0: 8 sqrt(m) 2^-24, reading Z14)")
a = ap.parse_args()
cfg = ts.CONFIGS[a.cfg]
b = ts.gen_batch(cfg, 0, a.batch)
s = T.TiltSolver(0, max_batch=a.batch, max_m=cfg.m, max_n=cfg.n, max_p=cfg.p, max_image_elems=b["images"].size)
prm = T.default_params(fixed_inner_iters=a.inner, fixed_outer_iters=a.outer, max_inner=max(a.inner, 1),
                       max_outer=max(a.outer, 1), win_h=cfg.m, win_w=cfg.n, kernel_path=a.path, ns_period=a.ns,
                       jacobi_tol=a.jtol, **({"jacobi_max_sweeps": a.max_sweeps} if a.max_sweeps else {}))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(a.reps):
    ev0.record()
    out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    ev1.record()
    torch.cuda.synchronize()
rep = T.reports_to_numpy(out["rep"])
ms = ev0.elapsed_time(ev1)
it = rep["inner_iters"].sum()
sw = rep["jacobi_sweeps"].sum()
m, n, p = cfg.m, cfg.n, cfg.p
fl = it * (8 * p * m * n + 20 * m * n + 4 * m * n * n + 4 * n ** 3 / max(1, a.ns)) + sw * n * (n - 1) / 2 * (12 * m + 6 * n)
rot = rep["jacobi_rotations"].sum()
pairs = sw * n * (n - 1) / 2
print(f"path={a.path} ns={a.ns} cfg={a.cfg} batch={a.batch} inner={a.inner} outer={a.outer}: {ms:.3f} ms, {it} iters, {sw/it:.2f} sweeps/iter, "
      f"{rot/max(pairs,1):.3f} rotations/pair-check, {it/ms*1e3:.0f} iters/s, {fl/ms/1e9:.2f} TFLOP/s (model)")
