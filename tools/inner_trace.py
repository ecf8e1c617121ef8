"""Inner-loop trace of one patch's first outer iteration: GPU (mu, crit1, crit2, rho per LADMAP
iteration) against the fp64 oracle's, to see why an fp32 inner loop misses Cond1 & Cond2 and runs to
max_inner where the oracle stops (SURVEY §8(c) protocol 3 diagnostics).
Usage: python tools/inner_trace.py --patch 0 [--ns 1] [--tol-scale 0.1]"""
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
    ap.add_argument("--patch", type=int, default=0)
    ap.add_argument("--outer", type=int, default=1)
    ap.add_argument("--variants", default="default;ns=1;tol=0.1;ns=1,tol=0.1")
    args = ap.parse_args()
    import torch
    import paper_1205_5351_b200 as T
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, args.patch, 1)
    r = O.tilt(b["images"][0], b["boxes"][0], b["tau0"][0], cfg.kind,
               O.Params(fixed_outer_iters=args.outer, max_outer=args.outer))
    tr = r["traces"][args.outer - 1]
    print(json.dumps({"side": "oracle", "iters": len(tr), "mu_last": tr[-1][0], "crit1_last": tr[-1][1],
                      "crit2_last": tr[-1][2],
                      "tail": [(round(t[0], 1), float(f"{t[1]:.3e}"), float(f"{t[2]:.3e}"), t[3]) for t in tr[-8:]]}))
    s = T.TiltSolver(0, max_batch=4, max_m=64, max_n=64, max_p=8)
    for v in args.variants.split(";"):
        kw = {}
        for item in v.split(","):
            if item.startswith("ns="):
                kw["ns_period"] = int(item[3:])
            if item.startswith("tol="):
                kw["jacobi_tol"] = float(item[4:]) * 8 * np.sqrt(cfg.m) * 2.0 ** -24
        prm = T.default_params(fixed_outer_iters=args.outer, max_outer=args.outer, **kw)
        trace = torch.full((1, args.outer, prm.max_inner, 4), float("nan"), device="cuda")
        prm.trace = trace.data_ptr()
        out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
        t = trace[0, args.outer - 1].cpu().numpy()
        k = int(np.sum(np.isfinite(t[:, 0])))
        rep = T.reports_to_numpy(out["rep"])[0]
        c2 = t[:k, 2]
        print(json.dumps({"side": "gpu", "variant": v, "iters": k, "sweeps_per_svt": float(rep["jacobi_sweeps"]) / max(1, int(rep["inner_iters"])),
                          "mu_last": float(t[k - 1, 0]), "crit1_min": float(np.nanmin(t[:k, 1])),
                          "crit2_min_after_500": float(np.nanmin(c2[500:])) if k > 500 else None,
                          "tail": [(round(float(x[0]), 1), float(f"{x[1]:.3e}"), float(f"{x[2]:.3e}"), float(x[3])) for x in t[max(0, k - 8):k]],
                          "at_oracle_stop": [(round(float(x[0]), 1), float(f"{x[1]:.3e}"), float(f"{x[2]:.3e}")) for x in t[len(tr) - 3:len(tr) + 3]]}))


if __name__ == "__main__":
    main()
