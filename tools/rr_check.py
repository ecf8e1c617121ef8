"""Register-resident vs shared-memory Jacobi layout (tilt_params.jacobi_layout 0 / 1) on the same
patches: fixed-count solves, max |A|, |E|, |tau| differences and per-layout counts; then the
free-running bench-shaped solve on both layouts (converged fraction, iterations, time)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--free", type=int, default=1024)
a = ap.parse_args()
cfg = ts.CONFIGS[a.cfg]
b = ts.gen_batch(cfg, 0, max(a.batch, a.free))
s = T.TiltSolver(0, max_batch=max(a.batch, a.free), max_m=cfg.m, max_n=cfg.n, max_p=cfg.p,
                 max_image_elems=b["images"].size)
for fo, fi in ((1, 1), (1, 5), (2, 20)):
    outs = []
    for jl in (0, 1):
        prm = T.default_params(fixed_inner_iters=fi, fixed_outer_iters=fo, max_inner=fi, max_outer=fo,
                               win_h=cfg.m, win_w=cfg.n, jacobi_layout=jl)
        sl = slice(0, a.batch)
        o = s.solve(b["images"], b["patch_image"][sl], b["boxes"][sl], b["tau0"][sl], cfg.kind, prm)
        outs.append(o)
    r0, r1 = (T.reports_to_numpy(o["rep"]) for o in outs)
    d = {k: float((outs[0][k] - outs[1][k]).abs().max()) for k in ("A", "E", "tau")}
    sc = {k: float(outs[1][k].abs().max()) for k in ("A", "E")}
    print(f"fixed outer={fo} inner={fi}: max|diff| A {d['A']:.3e} (|A| {sc['A']:.2e}) E {d['E']:.3e} tau {d['tau']:.3e}; "
          f"sweeps {r0['jacobi_sweeps'].sum()} vs {r1['jacobi_sweeps'].sum()}, rotations "
          f"{r0['jacobi_rotations'].sum()} vs {r1['jacobi_rotations'].sum()}, status equal "
          f"{bool((r0['status'] == r1['status']).all())}", flush=True)
for jl in (0, 1):
    prm = T.default_params(win_h=cfg.m, win_w=cfg.n, jacobi_layout=jl)
    sl = slice(0, a.free)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = s.solve(b["images"], b["patch_image"][sl], b["boxes"][sl], b["tau0"][sl], cfg.kind, prm)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    r = T.reports_to_numpy(o["rep"])
    conv = int((r["status"] == 0).sum())
    print(f"free-running jl={jl}: {dt:.3f} s, {conv}/{a.free} converged, {r['inner_iters'].sum()} inner iters "
          f"({r['inner_iters'].sum() / dt / 1e6:.3f} M it/s), {r['jacobi_sweeps'].sum() / r['inner_iters'].sum():.2f} sweeps/it",
          flush=True)
