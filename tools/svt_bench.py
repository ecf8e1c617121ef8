"""Micro-benchmark of the SVT kernels alone (tilt_svt_batch): B random m x n low-rank + noise
matrices, cold V; prints time, sweeps and Jacobi pair-rotations per second for the
warp-per-patch (path 0) and CTA-per-patch (path 1) kernels.
Usage: python tools/svt_bench.py [--m 50] [--n 50] [--batch 2368] [--reps 3] [--paths 0,1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_5351_b200 as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--n", type=int, default=50)
ap.add_argument("--batch", type=int, default=2368)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--paths", default="0,1")
a = ap.parse_args()
rng = np.random.default_rng(0)
B, m, n = a.batch, a.m, a.n
U = rng.normal(size=(B, m, 5)) @ rng.normal(size=(B, 5, n)) + 0.05 * rng.normal(size=(B, m, n))
M = torch.as_tensor(U.astype(np.float32), device="cuda")
eps = np.full(B, 0.5, np.float32)
s = T.TiltSolver(0, max_batch=B, max_m=m, max_n=n, max_p=8)
for path in [int(p) for p in a.paths.split(",")]:
    out = s.svt(M, eps, path=path)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(a.reps):
        e0.record()
        out = s.svt(M, eps, path=path)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    sw = out["sweeps"].double().mean().item()
    pairs = B * sw * n * (n - 1) / 2
    print(f"path={path} m={m} n={n} B={B}: {t:.3f} ms, {sw:.2f} sweeps, {pairs / t / 1e6:.3f} G pair-steps/s, "
          f"{t * 1e3 / (sw * (n - 1)):.2f} us per round (whole batch)", flush=True)
