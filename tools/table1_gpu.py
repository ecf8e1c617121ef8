"""Table 1 of the paper on the B200: the inner loop alone on random data (reading Z20),
ADM baseline vs LADMAP, batched. For each size: mean iterations, mean objective and GPU time per
problem (batch of B independent problems in one tilt_inner_batch call, CUDA events), next to the
paper's MATLAB/Xeon numbers (context only, another machine).
Usage: python tools/table1_gpu.py [--sizes 10,50,100] [--batch 1024] [--trials 10]"""
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

PAPER = {10: {"adm": (1.98e-5, 49.2, 6.4836), "ladmap": (7.49e-6, 20.4, 6.4814)},
         50: {"adm": (0.00112, 51.5, 76.6508), "ladmap": (0.00054, 21.2, 76.6468)},
         100: {"adm": (0.00538, 51.1, 217.001), "ladmap": (0.00252, 22.2, 216.985)}}

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="10,50,100")
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--trials", type=int, default=10, help="instances whose mean is reported (the paper's 10)")
a = ap.parse_args()
rows = []
for n in [int(x) for x in a.sizes.split(",")]:
    B = a.batch if n <= 64 else min(a.batch, 256)
    insts = [ts.table1_instance(n, 6, s) for s in range(B)]
    D = torch.as_tensor(np.stack([i["D"] for i in insts]).astype(np.float32), device="cuda")
    J = torch.as_tensor(np.stack([i["J"] for i in insts]).astype(np.float32), device="cuda")
    s = T.TiltSolver(0, max_batch=B, max_m=n, max_n=n, max_p=6)
    for name, solver_id in (("adm", 1), ("ladmap", 0)):
        prm = T.default_params(inner_solver=solver_id)
        s.inner(D, J, params=prm)  # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = s.inner(D, J, params=prm)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rep = out["rep"]
        row = {"n": n, "solver": name, "batch": B, "gpu_ms_batch": ms, "gpu_s_per_problem": ms / 1e3 / B,
               "iters_mean_first_trials": float(np.mean(rep["inner_iters"][:a.trials])),
               "objective_mean_first_trials": float(np.mean(rep["objective"][:a.trials])),
               "iters_mean_batch": float(np.mean(rep["inner_iters"])),
               "converged": float(np.mean(rep["status"] == T.CONVERGED))}
        if n in PAPER:
            t, it, obj = PAPER[n][name]
            row.update({"paper_time_s": t, "paper_iters": it, "paper_objective": obj})
        rows.append(row)
        print(json.dumps(row), flush=True)
    s.close()
