"""Inner loop (Table 1 data, reading Z20) on the CTA-per-patch kernels vs the multi-CTA path over
window sizes, at a fixed batch: the evidence behind kernel_path = 0's switch at 128 x 128.
Usage: python tools/inner_paths.py [--sizes 64,100,128,160,200,256] [--batch 64]"""
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
ap.add_argument("--sizes", default="64,100,128,160,200,256")
ap.add_argument("--batch", type=int, default=64)
a = ap.parse_args()
sizes = [int(x) for x in a.sizes.split(",")]
s = T.TiltSolver(0, max_batch=a.batch, max_m=max(sizes), max_n=max(sizes), max_p=8)
for n in sizes:
    insts = [ts.table1_instance(n, 6, k) for k in range(a.batch)]
    D = torch.as_tensor(np.stack([i["D"] for i in insts]).astype(np.float32), device="cuda")
    J = torch.as_tensor(np.stack([i["J"] for i in insts]).astype(np.float32), device="cuda")
    row = {"size": n, "batch": a.batch}
    for path in (1, 3):
        prm = T.default_params(kernel_path=path)
        s.inner(D, J, params=prm)  # warm-up (workspace allocation, cuBLAS)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = s.inner(D, J, params=prm)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        rep = out["rep"]
        row[f"path{path}_s"] = t
        row[f"path{path}_iters_mean"] = float(rep["inner_iters"].mean())
        row[f"path{path}_objective_mean"] = float(rep["objective"].mean())
    row["speedup_multi_cta"] = row["path1_s"] / row["path3_s"]
    print(json.dumps(row), flush=True)
