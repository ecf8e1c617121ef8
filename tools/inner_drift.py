"""Fixed-count parity far into one inner loop: A, E of the GPU after K LADMAP iterations (the oracle's
rho decisions replayed, Z21) against the oracle's, K up to beyond the oracle's own stop -- does the
fp32 iterate drift from the fp64 one at large mu? (protocol-3 diagnostics; config-2 patch, first
outer iteration)."""
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
    ap.add_argument("--patch", type=int, default=21)
    ap.add_argument("--ks", default="20,50,100,200,300,400,450,600,800")
    args = ap.parse_args()
    import torch
    import paper_1205_5351_b200 as T
    cfg = ts.CONFIGS[2]
    b = ts.gen_batch(cfg, args.patch, 1)
    s = T.TiltSolver(0, max_batch=4, max_m=64, max_n=64, max_p=8)
    for K in [int(x) for x in args.ks.split(",")]:
        r = O.tilt(b["images"][0], b["boxes"][0], b["tau0"][0], cfg.kind,
                   O.Params(fixed_outer_iters=1, max_outer=1, fixed_inner_iters=K, max_inner=K))
        bits = np.zeros((1, 1, K), np.uint8)
        bits[0, 0, :] = [t[3] for t in r["traces"][0]]
        rr = torch.as_tensor(bits, device="cuda")
        prm = T.default_params(fixed_outer_iters=1, max_outer=1, fixed_inner_iters=K, max_inner=K)
        prm.rho_replay = rr.data_ptr()
        out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
        a = out["A"][0].double().cpu().numpy()
        e = out["E"][0].double().cpu().numpy()
        print(json.dumps({"K": K, "mu": r["traces"][0][-1][0], "relA": float(np.linalg.norm(a - r["A"]) / np.linalg.norm(r["A"])),
                          "relE": float(np.linalg.norm(e - r["E"]) / np.linalg.norm(r["E"])),
                          "crit2_oracle": r["traces"][0][-1][2]}), flush=True)


if __name__ == "__main__":
    main()
