"""Isolate a failure of the register-resident Jacobi: one solve per process (batch, fixed outer/inner,
ctas_per_sm, jacobi_layout), printing ok / the error."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys; sys.path.insert(0, %r)
import torch, paper_1205_5351_b200 as T, tilt_synth as ts
B, fo, fi, cps, jl = %d, %d, %d, %d, %d
cfg = ts.CONFIGS[2]; b = ts.gen_batch(cfg, 0, B)
s = T.TiltSolver(0, max_batch=B, max_m=cfg.m, max_n=cfg.n, max_p=cfg.p, max_image_elems=b["images"].size)
kw = dict(fixed_inner_iters=fi, fixed_outer_iters=fo, max_inner=fi, max_outer=fo) if fi > 0 else {}
prm = T.default_params(win_h=cfg.m, win_w=cfg.n, ctas_per_sm=cps, jacobi_layout=jl, **kw)
o = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
torch.cuda.synchronize()
r = T.reports_to_numpy(o["rep"])
print("ok", int(r["inner_iters"].sum()), int(r["jacobi_sweeps"].sum()))
'''
cases = [(64, 1, 1, 0, 0), (592, 1, 1, 0, 0), (592, 1, 1, 1, 0), (148, 1, 1, 0, 0), (296, 1, 1, 0, 0),
         (592, 1, 30, 1, 0), (64, 1, 30, 0, 0), (64, 2, 60, 0, 0), (592, 1, 1, 2, 0), (64, 0, 0, 0, 0),
         (592, 1, 1, 0, 1)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in c.split(",")) for c in sys.argv[1:]]
for c in cases:
    try:
        p = subprocess.run([sys.executable, "-c", CASE % ((ROOT,) + c)], capture_output=True, text=True, timeout=300)
        out = (p.stdout.strip().splitlines() or [""])[-1]
        err = [l for l in p.stderr.splitlines() if "Error" in l or "error" in l][-1:] 
        print(c, out, err, flush=True)
    except subprocess.TimeoutExpired:
        print(c, "timeout", flush=True)
