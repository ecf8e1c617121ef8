"""Config 2 (1024 x 50x50 homography) makespan vs CTAs per SM, and where the longest patches sit in
the queue (the batch tail). Usage: python tools/tail_probe.py [--cps 4,3,2]"""
import argparse
import json
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
ap.add_argument("--cps", default="4,3,2")
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
cfg = ts.CONFIGS[a.config]
B = cfg.batch
b = bench.gen_shard(a.config, range(B))
s = T.TiltSolver(0, max_batch=B, max_m=cfg.m, max_n=cfg.n, max_p=cfg.p, max_image_elems=int(b["images"].size))
args = [torch.as_tensor(b["images"], device="cuda"), torch.arange(B, dtype=torch.int32, device="cuda"),
        torch.as_tensor(b["boxes"], device="cuda"), torch.as_tensor(b["tau0"], device="cuda")]
for cps in [int(c) for c in a.cps.split(",")]:
    prm = T.default_params(win_h=cfg.m, win_w=cfg.n, ctas_per_sm=cps)
    s.solve(*args, cfg.kind, prm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(*args, cfg.kind, prm, sync=False)
    e1.record()
    torch.cuda.synchronize()
    rep = T.reports_to_numpy(out["rep"])
    it = rep["inner_iters"]
    top = np.argsort(-it)[:5]
    print(json.dumps({"config": a.config, "ctas_per_sm": cps, "seconds": e0.elapsed_time(e1) / 1e3,
                      "total_inner": int(it.sum()), "top5_idx": top.tolist(), "top5_inner": it[top].tolist()}),
          flush=True)
