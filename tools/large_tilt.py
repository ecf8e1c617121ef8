"""Full Algorithm 1 on large windows (multi-CTA path): B synthetic patches of an m x m window
(affine, rank 2-3 textures, rotation +-10 deg, skew +-0.1, 5% corruption; tilt_synth recipe) solved
free-running by tilt_solve_batch; optionally config 4 (256 x 200x200) on both kernel families.
Usage: python tools/large_tilt.py [--sizes 300,500] [--batch 8] [--config4 0|1]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="300,500")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--config4", type=int, default=0)
ap.add_argument("--max-outer", type=int, default=50)
a = ap.parse_args()


def run(cfg, B, path, label):
    b = ts.gen_batch(cfg, 0, B)
    s = T.TiltSolver(0, max_batch=B, max_m=cfg.m, max_n=cfg.n, max_p=8, max_image_elems=int(b["images"].size))
    prm = T.default_params(kernel_path=path, max_outer=a.max_outer)
    imgs = torch.as_tensor(b["images"], device="cuda")
    args = (imgs, torch.as_tensor(b["patch_image"], device="cuda"), torch.as_tensor(b["boxes"], device="cuda"),
            torch.as_tensor(b["tau0"], device="cuda"), cfg.kind, prm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(*args)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    rep = T.reports_to_numpy(out["rep"])
    row = {"case": label, "window": f"{cfg.m}x{cfg.n}", "batch": B, "kernel_path": path, "seconds": t,
           "converged": int((rep["status"] == T.CONVERGED).sum()), "status": np.bincount(rep["status"], minlength=6).tolist(),
           "mean_outer": float(rep["outer_iters"].mean()), "mean_inner": float(rep["inner_iters"].mean()),
           "inner_iters_per_s": float(rep["inner_iters"].sum() / t),
           "sweeps_per_svt": float(rep["jacobi_sweeps"].sum() / max(1, rep["inner_iters"].sum()))}
    print(json.dumps(row), flush=True)
    s.close()


for m in [int(x) for x in a.sizes.split(",") if x]:
    cfg = ts.SynthConfig(90 + m // 100, a.batch, m, m, 0, 2, 3, 10.0, 0.1, 0.0, 0.05)
    run(cfg, a.batch, 3, f"synthetic {m}x{m}")
if a.config4:
    cfg = ts.CONFIGS[4]
    run(cfg, cfg.batch, 3, "config 4 (multi-CTA)")
    run(cfg, cfg.batch, 1, "config 4 (CTA)")
