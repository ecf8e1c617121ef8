"""Profiling driver of the multi-CTA path: one tilt_inner_batch call on Table 1 data (reading Z20)
at size n with B trials and a fixed inner iteration count. Prints the event time.
Usage: python tools/lp_prof.py [--n 1000] [--batch 1] [--inner 2] [--reps 1]"""
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
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--inner", type=int, default=2)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
insts = [ts.table1_instance(a.n, 6, k) for k in range(a.batch)]
D = torch.as_tensor(np.stack([i["D"] for i in insts]).astype(np.float32), device="cuda")
J = torch.as_tensor(np.stack([i["J"] for i in insts]).astype(np.float32), device="cuda")
s = T.TiltSolver(0, max_batch=a.batch, max_m=a.n, max_n=a.n, max_p=8)
prm = T.default_params(kernel_path=3, fixed_inner_iters=a.inner, max_inner=max(a.inner, 1))
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.inner(D, J, params=prm)
    e1.record()
    torch.cuda.synchronize()
    rep = out["rep"]
    print(f"n={a.n} B={a.batch} inner={a.inner}: {e0.elapsed_time(e1):.2f} ms, sweeps/SVT "
          f"{rep['jacobi_sweeps'].sum() / max(1, rep['inner_iters'].sum()):.2f}, aux sweeps {rep['aux_sweeps'].mean():.1f}")
