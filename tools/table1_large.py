"""Table 1 at its large sizes on the multi-CTA path: 10 random trials per size
(reading Z20), solved as one batched tilt_inner_batch call and, for latency, one trial alone; prints
iterations, objective and time per trial next to the paper's LADMAP columns (MATLAB, Xeon E5540).
Usage: python tools/table1_large.py [--sizes 300,500,1000] [--trials 10] [--out FILE]"""
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

PAPER = {  # size: (time s, #iter, objective) of LADMAP, ADM, LADMAP+SVDWS -- P:956-970
    100: ((0.00252, 22.2, 216.985), (0.00538, 51.1, 217.001), (0.00225, 22.9, 216.987)),
    300: ((0.10501, 21.9, 1123.67), (0.1859, 50, 1123.66), (0.08792, 22.9, 1123.70)),
    500: ((0.6574, 22, 2419.63), (1.3802, 50, 2420.41), (0.5343, 21, 2420.28)),
    1000: ((25.8139, 23, 6844.14), (53.0936, 50, 6844.82), (18.5953, 23, 6845.32)),
}

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="300,500,1000")
ap.add_argument("--trials", type=int, default=10)
ap.add_argument("--p", type=int, default=6)
ap.add_argument("--out", default="")
ap.add_argument("--svd-mode", type=int, default=0, help="tilt_params.svd_mode (1: LADMAP+SVDWS, Alg. 2)")
ap.add_argument("--gate", type=float, default=2e-5, help="tilt_params.svd_ws_gate (eps_svd / ||D||_F)")
ap.add_argument("--adm", type=int, default=0, help="1: the ADM baseline (tilt_params.inner_solver = 1)")
ap.add_argument("--eps2-scale", type=float, default=0.0,
                help="> 0: eps2 = scale * 50 / n (Cond2 is not scale-invariant, Z7; the paper tunes eps2 per size)")
a = ap.parse_args()
sizes = [int(x) for x in a.sizes.split(",")]
nmax = max(sizes)
s = T.TiltSolver(0, max_batch=a.trials, max_m=nmax, max_n=nmax, max_p=8)
rows = []
for n in sizes:
    insts = [ts.table1_instance(n, a.p, k) for k in range(a.trials)]
    D = torch.as_tensor(np.stack([i["D"] for i in insts]).astype(np.float32), device="cuda")
    J = torch.as_tensor(np.stack([i["J"] for i in insts]).astype(np.float32), device="cuda")
    prm = T.default_params(kernel_path=3, svd_mode=a.svd_mode, svd_ws_gate=a.gate, inner_solver=a.adm)
    if a.eps2_scale > 0:
        prm.eps2 = a.eps2_scale * 50.0 / n
    s.inner(D[:1], J[:1], params=prm)  # warm-up (workspace, cuBLAS)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    one = s.inner(D[:1], J[:1], params=prm)
    e1.record()
    torch.cuda.synchronize()
    t_one = e0.elapsed_time(e1) / 1e3
    e0.record()
    out = s.inner(D, J, params=prm)
    e1.record()
    torch.cuda.synchronize()
    t_all = e0.elapsed_time(e1) / 1e3
    rep = out["rep"]
    it, sw = rep["inner_iters"], rep["jacobi_sweeps"]
    lad = PAPER.get(n, ((None,) * 3,) * 3)[1 if a.adm else (2 if a.svd_mode == 1 else 0)]
    row = {"size": n, "trials": a.trials, "p": a.p, "solver": "adm" if a.adm else "ladmap", "svd_mode": a.svd_mode, "eps2": float(prm.eps2),
           "gate": a.gate,
           "warm_steps_mean": float(rep["svd_warm_steps"].mean()), "iters_mean": float(it.mean()),
           "objective_mean": float(rep["objective"].mean()), "sweeps_per_svt": float(sw.sum() / it.sum()),
           "converged": int((rep["status"] == T.CONVERGED).sum()),
           "time_one_trial_s": t_one, "time_batch_s": t_all, "time_per_trial_batched_s": t_all / a.trials,
           "one_trial_iters": int(one["rep"]["inner_iters"][0]),
           "paper_time_s": lad[0], "paper_iters": lad[1], "paper_objective": lad[2]}
    if lad[0]:
        row["speedup_one_trial_vs_paper"] = lad[0] / t_one
        row["speedup_batched_vs_paper"] = lad[0] / (t_all / a.trials)
    rows.append(row)
    print(json.dumps(row), flush=True)
if a.out:
    with open(a.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
