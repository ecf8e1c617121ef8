"""Fig. 2 (range of convergence) as one batched GPU call per solver: the
checker-board deformed by A(theta, t) = R(theta)[[1, t], [0, 1]] on the paper's grid (theta in
[0, pi/6] step pi/60, t in [0, 1] step 0.05), TILT from tau0 = I with the LADMAP inner loop (the
paper's) and with the ADM baseline; success = tilt_synth.metrics.rectified (reading Z25).
Prints both success maps (rows theta, columns t) and the counts; --oracle K re-runs K cells on the
fp64 oracle and reports agreement. Usage: python tools/range_of_convergence.py [--m 32] [--oracle 6]"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402
from tilt_synth.metrics import rectified  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--square", type=int, default=8)
ap.add_argument("--oracle", type=int, default=0)
ap.add_argument("--json", default="")
a = ap.parse_args()
g = ts.convergence_grid(a.m, a.square)
B = g["images"].shape[0]
nt, ns = len(g["thetas"]), len(g["skews"])
s = T.TiltSolver(0, max_batch=B, max_m=a.m, max_n=a.m, max_p=6, max_image_elems=int(g["images"].size))
result = {"m": a.m, "square_px": a.square, "thetas_deg": [math.degrees(x) for x in g["thetas"]], "skews": g["skews"]}
for name, sid in (("ladmap", 0), ("adm", 1)):
    prm = T.default_params(inner_solver=sid)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(g["images"], g["patch_image"], g["boxes"], g["tau0"], T.AFFINE, prm)
    e1.record()
    torch.cuda.synchronize()
    tau = out["tau"].double().cpu().numpy()
    ok = np.array([rectified(tau[k], g["tau_g"][k]) for k in range(B)]).reshape(nt, ns)
    result[name] = {"success": ok.astype(int).tolist(), "count": int(ok.sum()), "ms": e0.elapsed_time(e1)}
    print(f"{name}: {int(ok.sum())}/{B} rectified, one batched solve {e0.elapsed_time(e1):.1f} ms")
    print("      t=" + "".join(f"{t:5.2f}"[1:] if t < 1 else " 1.0" for t in g["skews"]))
    for i, th in enumerate(g["thetas"]):
        print(f"{math.degrees(th):5.1f}   " + "".join("   #" if v else "   ." for v in ok[i]))
lad, adm = np.array(result["ladmap"]["success"]), np.array(result["adm"]["success"])
result["adm_not_ladmap"] = int(np.sum((adm == 1) & (lad == 0)))
result["ladmap_not_adm"] = int(np.sum((lad == 1) & (adm == 0)))
print(f"cells rectified by ADM but not LADMAP: {result['adm_not_ladmap']}; by LADMAP but not ADM: {result['ladmap_not_adm']}")
if a.oracle > 0:
    import oracle as O
    rng = np.random.default_rng(0)
    agree = 0
    cells = rng.choice(B, size=a.oracle, replace=False)
    prm = T.default_params()
    out = s.solve(g["images"], g["patch_image"], g["boxes"], g["tau0"], T.AFFINE, prm)
    tau = out["tau"].double().cpu().numpy()
    for k in cells:
        t0 = time.time()
        r = O.tilt(g["images"][k], g["boxes"][k], g["tau0"][k], O.AFFINE)
        so, sg = rectified(r["tau"], g["tau_g"][k]), rectified(tau[k], g["tau_g"][k])
        agree += so == sg
        print(f"oracle cell {k}: oracle rectified={so} gpu rectified={sg} max|dtau|={np.max(np.abs(r['tau'] - tau[k])):.2e} "
              f"({time.time() - t0:.1f}s)")
    result["oracle_agreement"] = f"{agree}/{a.oracle}"
if a.json:
    json.dump(result, open(a.json, "w"))
