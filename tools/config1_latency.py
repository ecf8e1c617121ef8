"""Config 1 (one 32x32 affine patch, BASELINE.json configs[0]) solve latency on the CTA-per-patch
and warp-per-patch kernels. Usage: python tools/config1_latency.py"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1205_5351_b200 as T, tilt_synth as ts
cfg = ts.CONFIGS[1]
b = ts.gen_batch(cfg, 0, 1)
s = T.TiltSolver(0, max_batch=4, max_m=32, max_n=32, max_p=6, max_image_elems=int(b["images"].size))
for path in (1, 2):
    prm = T.default_params(kernel_path=path, win_h=32, win_w=32)
    s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts_ = []
    for _ in range(3):
        e0.record(); out = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm, sync=False); e1.record(); torch.cuda.synchronize()
        ts_.append(e0.elapsed_time(e1))
    rep = T.reports_to_numpy(out["rep"])[0]
    print(f"config 1 latency path={path}: {min(ts_):.1f} ms, status {rep['status']}, outer {rep['outer_iters']}, inner {rep['inner_iters']}, {rep['inner_iters']/min(ts_)*1e3:.0f} iter/s")
