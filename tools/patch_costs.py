"""Per-patch work of the bench batch (config 2, 1024 patches): inner iterations, outer iterations and
status of every patch, for the scheduling analysis (tail effect). Usage: python tools/patch_costs.py OUT.npz"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402

cfg = ts.CONFIGS[2]
b = bench.gen_shard(2, 0, 1024)
s = T.TiltSolver(0, max_batch=1024, max_m=50, max_n=50, max_p=8, max_image_elems=int(b["images"].size))
out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, T.default_params(win_h=50, win_w=50))
rep = T.reports_to_numpy(out["rep"])
np.savez(sys.argv[1], inner=rep["inner_iters"], outer=rep["outer_iters"], status=rep["status"],
         sweeps=rep["jacobi_sweeps"])
print("max inner", rep["inner_iters"].max(), "argmax", int(rep["inner_iters"].argmax()), "mean", rep["inner_iters"].mean())
