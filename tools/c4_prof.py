"""Config 4 on the multi-CTA path with fixed counts (for a launch list / host-overhead split):
B patches 200x200 affine, fixed_outer_iters outer x fixed_inner_iters inner iterations.
Prints the CUDA-event time of the call and the launches it issued.
Usage: python tools/c4_prof.py [--batch 256] [--outer 1] [--inner 30]"""
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
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--outer", type=int, default=1)
ap.add_argument("--inner", type=int, default=30)
a = ap.parse_args()
cfg = ts.CONFIGS[4]
b = bench.gen_shard(4, range(a.batch))
s = T.TiltSolver(0, max_batch=a.batch, max_m=cfg.m, max_n=cfg.n, max_p=cfg.p)
prm = T.default_params(win_h=cfg.m, win_w=cfg.n, fixed_outer_iters=a.outer, max_outer=a.outer,
                       fixed_inner_iters=a.inner, max_inner=a.inner)
args = (torch.as_tensor(b["images"], device="cuda"), torch.arange(a.batch, dtype=torch.int32, device="cuda"),
        torch.as_tensor(b["boxes"], device="cuda"), torch.as_tensor(b["tau0"], device="cuda"), cfg.kind, prm)
s.solve(*args)
for r in range(2):
    l0 = s.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(*args, sync=False)
    e1.record()
    torch.cuda.synchronize()
    rep = T.reports_to_numpy(out["rep"])
    print(f"config 4 x{a.batch}, {a.outer} outer x {a.inner} inner: {e0.elapsed_time(e1):.1f} ms, "
          f"{s.launches - l0} launches, {float(np.mean(rep['jacobi_sweeps'])) / max(1, a.inner * a.outer):.2f} sweeps/SVT",
          flush=True)
