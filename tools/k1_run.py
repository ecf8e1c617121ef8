"""K1 (warp/Jacobian) HBM roofline over the first N patches of the bench workload (config 5), as
bench.py measures it (cold L2 before each launch, median of 20). Usage: python tools/k1_run.py [N]"""
import sys, os
sys.path.insert(0, os.getcwd())
import bench, json, numpy as np, torch
import paper_1205_5351_b200 as T, tilt_synth as ts
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = ts.CONFIGS[5]
b = bench.gen_shard(5, range(N))
images = torch.as_tensor(b["images"], device="cuda"); pi = torch.arange(N, dtype=torch.int32, device="cuda")
boxes = torch.as_tensor(b["boxes"], device="cuda"); tau0 = torch.as_tensor(b["tau0"], device="cuda")
s = T.TiltSolver(0, max_batch=N, max_m=50, max_n=50, max_p=8, max_image_elems=int(images.numel()))
print(json.dumps(bench.k1_roofline(s, images, pi, boxes, tau0, cfg.kind, 50, 50, 8, bench._peaks())))
