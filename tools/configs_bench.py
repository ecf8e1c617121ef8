"""Throughput of the hot entry on every BASELINE.json config (synthetic, tilt_synth seeds), one GPU:
converged patches/s, LADMAP iterations/s and the FP32 model rate per config. Config 3 uses the
2-level pyramid (reading Z18). Batches: the config's own (config 5 = config 2's shape: its 65536
patches are the multi-GPU workload; here 8192 on one GPU).
Usage: python tools/configs_bench.py [--configs 1,2,3,4,5] [--cap 8192]"""
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
ap.add_argument("--configs", default="1,2,3,4,5")
ap.add_argument("--cap", type=int, default=8192)
ap.add_argument("--pyramid-warm", type=int, default=0, help="tilt_params.pyramid_warm (config 3; reading Z26)")
ap.add_argument("--kernel-path", type=int, default=0, help="tilt_params.kernel_path (0 auto, 1 CTA, 3 multi-CTA)")
a = ap.parse_args()
for cid in [int(c) for c in a.configs.split(",")]:
    cfg = ts.CONFIGS[cid]
    B = min(cfg.batch, a.cap)
    b = bench.gen_shard(cid, range(B))
    b["patch_image"] = np.arange(B, dtype=np.int32)
    m, n, p = cfg.m, cfg.n, cfg.p
    s = T.TiltSolver(0, max_batch=B, max_m=m, max_n=n, max_p=p, max_image_elems=int(b["images"].size))
    prm = T.default_params(win_h=m, win_w=n, pyramid_levels=cfg.pyramid_levels, pyramid_warm=a.pyramid_warm,
                           kernel_path=a.kernel_path)
    imgs = torch.as_tensor(b["images"], device="cuda")
    args = (imgs, torch.as_tensor(b["patch_image"], device="cuda"), torch.as_tensor(b["boxes"], device="cuda"),
            torch.as_tensor(b["tau0"], device="cuda"), cfg.kind, prm)
    s.solve(*args)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(*args, sync=False)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    rep = T.reports_to_numpy(out["rep"])
    conv = int(np.sum(rep["status"] == T.CONVERGED))
    it = float(np.sum(rep["inner_iters"]))
    row = {"config": cid, "batch": B, "window": f"{m}x{n}", "p": p, "pyramid": cfg.pyramid_levels,
           "pyramid_warm": a.pyramid_warm, "kernel_path": a.kernel_path, "seconds": t,
           "converged_patches_per_s": conv / t, "converged_fraction": conv / B, "inner_iters_per_s": it / t,
           "mean_inner_iters": it / B, "sweeps_per_svt": float(np.sum(rep["jacobi_sweeps"]) / max(it, 1)),
           "max_inner_iters_patch": int(np.max(rep["inner_iters"])),
           "model_tflops": bench.flops_model(rep, m, n, p, int(prm.ns_period)) / t / 1e12}
    print(json.dumps(row), flush=True)
    s.close()
