"""Fig. 4 (robustness under corruption) as batched GPU solves: N synthetic
rank-3 textures rotated by 10 degrees, a fraction f of canvas pixels replaced by U[0,1]
(f = 0, 0.1, ..., 1.0), TILT from tau0 = I with LADMAP and with the ADM baseline; success =
tilt_synth.metrics.rectified. Prints success rates per level.
Usage: python tools/corruption_sweep.py [--textures 32] [--m 32]"""
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
from tilt_synth.metrics import rectified  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--textures", type=int, default=32)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--json", default="")
a = ap.parse_args()
levels = [round(0.1 * k, 1) for k in range(11)]
cases = [ts.corruption_case(i, f, a.m) for f in levels for i in range(a.textures)]
imgs = np.stack([c["canvas"] for c in cases])
boxes = np.stack([c["box"] for c in cases])
tau0 = np.stack([c["tau0"] for c in cases])
tau_g = np.stack([c["tau_g"] for c in cases])
B = len(cases)
s = T.TiltSolver(0, max_batch=B, max_m=a.m, max_n=a.m, max_p=6, max_image_elems=int(imgs.size))
res = {"levels": levels, "textures": a.textures}
for name, sid in (("ladmap", 0), ("adm", 1)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(imgs, np.arange(B, dtype=np.int32), boxes, tau0, T.AFFINE, T.default_params(inner_solver=sid))
    e1.record()
    torch.cuda.synchronize()
    tau = out["tau"].double().cpu().numpy()
    ok = np.array([rectified(tau[k], tau_g[k]) for k in range(B)]).reshape(len(levels), a.textures)
    res[name] = ok.mean(axis=1).tolist()
    print(f"{name} ({B} solves in one call, {e0.elapsed_time(e1):.0f} ms): " +
          " ".join(f"{f:.1f}:{r:.2f}" for f, r in zip(levels, ok.mean(axis=1))))
if a.json:
    json.dump(res, open(a.json, "w"))
