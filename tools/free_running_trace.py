"""Where do free-running GPU and oracle trajectories part? (SURVEY §8(c) protocol 3 diagnostics)

For config-2 patches: the fp64 oracle runs free (default tolerances) and records tau after every
outer iteration; the GPU runs with fixed_outer_iters = k for k = 1..n (its own rho decisions and
inner stops) and the max-abs tau difference per outer step is printed, with the inner-iteration
counts of each step on both sides.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import tilt_synth as ts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--patches", default="25,44,62,22,21,0,1")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_1205_5351_b200 as T
    cfg = ts.CONFIGS[2]
    s = T.TiltSolver(0, max_batch=64, max_m=64, max_n=64, max_p=8)
    rows = []
    for idx in [int(x) for x in args.patches.split(",")]:
        b = ts.gen_batch(cfg, idx, 1)
        r = O.tilt(b["images"][0], b["boxes"][0], b["tau0"][0], cfg.kind)
        n = max(1, r["outer_iters"])
        path = r["tau_path"]
        inner_or = [len(t) for t in r["traces"]]
        diffs, inner_gpu = [], []
        for k in range(1, n + 1):
            prm = T.default_params(fixed_outer_iters=k)
            out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
            rep = T.reports_to_numpy(out["rep"])[0]
            tau = out["tau"][0].double().cpu().numpy()
            diffs.append(float(np.max(np.abs(tau - path[k - 1]))))
            inner_gpu.append(int(rep["inner_iters"]))
        inner_gpu_step = np.diff([0] + inner_gpu).tolist()
        row = {"patch": idx, "outer": n, "dtau": diffs, "inner_oracle": inner_or, "inner_gpu": inner_gpu_step}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for row in rows:
                f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
