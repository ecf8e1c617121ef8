"""Small invocations of every kernel family: the CTA-per-patch solve (S32 and S64 classes), the
K1 warp, SVT, projector and inner entries, and the multi-CTA path (LADMAP and LADMAP+SVDWS with
the LU-solved Cayley step) -- a quick "everything launches and returns" check, and the program the
compute-sanitizer runs use (profiles/r02/sanitizer_*.log).
Usage: python tools/all_kernels_smoke.py [--only NAME]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_5351_b200 as T  # noqa: E402
import tilt_synth as ts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--only", default="")
a = ap.parse_args()


def run(name, fn):
    if a.only and a.only != name:
        return
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


s = T.TiltSolver(0, max_batch=4, max_m=128, max_n=128, max_p=8, max_image_elems=4 * 200 * 200)


def solve(cfg_id, path, K=3):
    cfg = ts.CONFIGS[cfg_id]
    b = ts.gen_batch(cfg, 0, 2)
    prm = T.default_params(fixed_inner_iters=K, fixed_outer_iters=2, max_inner=K, max_outer=2, kernel_path=path)
    s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)


run("solve_s32", lambda: solve(1, 1))
run("solve_s64", lambda: solve(2, 1))


def entries():
    b = ts.gen_batch(ts.CONFIGS[2], 0, 2)
    s.warp(b["images"], b["patch_image"], b["boxes"], b["tau0"], ts.CONFIGS[2].kind)
    rng = np.random.default_rng(0)
    M = rng.normal(size=(2, 50, 50)).astype(np.float32)
    s.svt(M, [0.1, 0.2])
    J = rng.normal(size=(2, 8, 50, 50)).astype(np.float32)
    s.project(J, M)
    inst = [ts.table1_instance(50, 6, k) for k in range(2)]
    s.inner(np.stack([i["D"] for i in inst]).astype(np.float32), np.stack([i["J"] for i in inst]).astype(np.float32),
            params=T.default_params(fixed_inner_iters=3, max_inner=3))


run("entries", entries)


def large(mode):
    inst = [ts.table1_instance(100, 6, k) for k in range(2)]
    D = np.stack([i["D"] for i in inst]).astype(np.float32)
    J = np.stack([i["J"] for i in inst]).astype(np.float32)
    s.inner(D, J, params=T.default_params(kernel_path=3, svd_mode=mode, svd_ws_gate=1e-3, fixed_inner_iters=6,
                                          max_inner=6))
    rng = np.random.default_rng(1)
    s.svt(rng.normal(size=(2, 70, 40)).astype(np.float32), [0.1, 0.1], path=3)


run("large", lambda: large(0))
run("large_svdws", lambda: large(1))
s.close()
