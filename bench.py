#!/usr/bin/env python
"""Benchmark of the batched TILT hot path (BASELINE.json metric: rectified patches/s (converged),
LADMAP inner iterations/s, % of FP32 / HBM roofline).

One *step* = one call of the hot entry ``tilt_solve_batch`` over one batch: Algorithm 1 for every
patch (warp/Jacobian -> orthonormalise -> LADMAP inner loop with warm Jacobi SVT -> dtau) until
each patch retires. Workload (N = 1): BASELINE.json configs[1] = config 2, 1024 patches 50x50
homography, seeded synthetic data (tilt_synth). For N > 1 (torchrun, one rank per GPU) each rank
solves its own 1024-patch shard of the same patch stream (config 5 = config 2 sharded; weak
scaling, no data-path collective); the tau/report gather to rank 0 runs after the timed region.

Prints one JSON line on rank 0. ``--impl reference`` times the fp64 oracle (oracle/) instead, on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import subprocess
import sys
import tempfile
import time

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")  # the oracle baseline runs one process per patch

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import tilt_synth as ts  # noqa: E402

PER_RANK_BATCH = 1024
CFG_ID = 2
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 148 SMs x 128 FP32 lanes x FMA x sm_max_mhz


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _gen_one(args):
    cfg_id, idx = args
    return ts.gen_patch(ts.CONFIGS[cfg_id], idx)


def gen_shard(cfg_id: int, start: int, count: int, workers: int = 0, indices=None) -> dict:
    workers = workers or min(16, os.cpu_count() or 1)
    if indices is not None:
        count = len(indices)
        jobs = [(cfg_id, int(i)) for i in indices]
    else:
        jobs = [(cfg_id, start + i) for i in range(count)]
    if workers > 1 and count > 8:
        with mp.get_context("fork").Pool(workers) as pool:
            pats = pool.map(_gen_one, jobs, chunksize=16)
    else:
        pats = [_gen_one(j) for j in jobs]
    return {
        "images": np.stack([p["canvas"] for p in pats]),
        "patch_image": np.arange(count, dtype=np.int32),
        "boxes": np.stack([p["box"] for p in pats]),
        "tau0": np.stack([p["tau0"] for p in pats]).astype(np.float32),
    }


def flops_per_launch(rep, m, n, p, ns_period: int = 4) -> float:
    """Algorithmic FLOPs (SURVEY.md §8(d) model) from the device counters of one launch:
    per LADMAP iteration 8pmn + 20mn + 4mn^2 + 4n^3/ns_period (the Newton-Schulz step on V runs
    after every ns_period-th SVT, tilt_params.ns_period), per Jacobi sweep n(n-1)/2 (12m + 6n)."""
    it = float(np.sum(rep["inner_iters"]))
    sw = float(np.sum(rep["jacobi_sweeps"]))
    return it * (8 * p * m * n + 20 * m * n + 4 * m * n * n + 4 * n ** 3 / max(1, ns_period)) + \
        sw * n * (n - 1) / 2 * (12 * m + 6 * n)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                for k, nm in enumerate(names):
                    if r[4 + k].strip().lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _oracle_job(args):
    import oracle as O
    image, box, tau0 = args
    return O.tilt(image, box, tau0, ts.HOMOGRAPHY)


def cpu_sample(batch: dict, count: int, cores: int) -> dict:
    """The fp64 oracle as it stands on the first ``count`` patches, one process per patch."""
    jobs = [(batch["images"][k], batch["boxes"][k], batch["tau0"][k].astype(np.float64)) for k in range(count)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(cores, count)) as pool:
        res = pool.map(_oracle_job, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    conv = sum(1 for r in res if r["status"] == 0)
    inner = sum(r["inner_iters"] for r in res)
    return {"seconds": dt, "converged": conv, "inner_iters": inner, "cores": min(cores, count), "count": count}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    batch = gen_shard(CFG_ID, 0, args.cpu_sample)
    cores = os.cpu_count() or 1
    vals, inners, secs = [], [], []
    for _ in range(args.warmup if args.ref_warmup else 0):
        cpu_sample(batch, args.cpu_sample, cores)
    for _ in range(args.steps):
        r = cpu_sample(batch, args.cpu_sample, cores)
        vals.append(r["converged"] / r["seconds"])
        inners.append(r["inner_iters"] / r["seconds"])
        secs.append(r["seconds"])
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "rectified patches/s (converged)", "value": value, "unit": "patches/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config 2 sample: first {args.cpu_sample} of 1024 patches 50x50 homography",
                   "global_batch": args.cpu_sample, "patch": "50x50", "transform": "homography"},
        "inner_iters_per_s": float(np.mean(inners)),
        "cpu_baseline": {"value": value, "unit": "patches/s", "cores": min(cores, args.cpu_sample), "kind": "oracle",
                         "sample": f"first {args.cpu_sample} patches of config 2, one process per patch"},
        "e2e": {"value": value, "unit": "patches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist
    import paper_1205_5351_b200 as T
    from paper_1205_5351_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = ts.CONFIGS[CFG_ID]
    B = args.batch
    m, n, p, kind = cfg.m, cfg.n, cfg.p, cfg.kind
    # rank r solves patches r, r + N, r + 2N, ... of the first N*B patches (interleaved shards)
    batch = gen_shard(CFG_ID, 0, B, indices=D.shard_indices(B * world, world, rank))
    images = torch.as_tensor(batch["images"], device=dev)
    patch_image = torch.as_tensor(batch["patch_image"], device=dev)
    boxes = torch.as_tensor(batch["boxes"], device=dev)
    tau0 = torch.as_tensor(batch["tau0"], device=dev)
    solver = T.TiltSolver(local_rank, max_batch=B, max_m=m, max_n=n, max_p=p,
                          max_image_elems=int(images.numel()))
    prm = T.default_params(win_h=m, win_w=n)
    out = {
        "tau": torch.empty((B, p), dtype=torch.float32, device=dev),
        "A": torch.empty((B, m, n), dtype=torch.float32, device=dev),
        "E": torch.empty((B, m, n), dtype=torch.float32, device=dev),
        "Y": None,
        "rep": torch.empty((B, T.solver._abi.REPORT_BYTES), dtype=torch.uint8, device=dev),
    }
    l2_flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        solver.solve(images, patch_image, boxes, tau0, kind, prm, out=out, sync=False)

    for _ in range(args.warmup):
        l2_flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = solver.launches
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for k in range(args.steps):
        l2_flush.zero_()  # inputs (41 MB) are smaller than L2: flush between steps
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    t_all1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = solver.launches - launches0
    clk = clocks.stop() if clocks else None
    elapsed = t_all0.elapsed_time(t_all1) / 1e3
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    rep = T.reports_to_numpy(out["rep"])
    conv = int(np.sum(rep["status"] == T.CONVERGED))
    inner = int(np.sum(rep["inner_iters"]))
    flops = flops_per_launch(rep, m, n, p, int(prm.ns_period))
    stats = torch.tensor([elapsed, float(conv), float(inner), flops, float(np.mean(kern_ms))], dtype=torch.float64,
                         device=dev)
    if world > 1:
        cdev = stats.device if dist.get_backend() == "nccl" else "cpu"  # gloo smoke test: host tensors
        tmax = stats[0:1].clone().to(cdev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tot = stats[1:4].clone().to(cdev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        elapsed = float(tmax.item())
        conv_all, inner_all, flops_all = (float(x) for x in tot.tolist())
    else:
        conv_all, inner_all, flops_all = float(conv), float(inner), flops
    # end to end through the host-buffer API on every rank (max time over ranks, summed patches)
    e2e_line = None
    if not args.no_e2e:
        if world > 1:
            dist.barrier()
        e2e_line = e2e(solver, batch, kind, prm, args)
        if world > 1:
            cdev = dev if dist.get_backend() == "nccl" else "cpu"
            red = torch.tensor([e2e_line["_seconds"]], dtype=torch.float64, device=cdev)
            dist.all_reduce(red, op=dist.ReduceOp.MAX)
            tot = torch.tensor([float(e2e_line["_conv"]), float(e2e_line["h2d_bytes_per_step"]),
                                float(e2e_line["d2h_bytes_per_step"])], dtype=torch.float64, device=cdev)
            dist.all_reduce(tot, op=dist.ReduceOp.SUM)
            e2e_line["_seconds"] = float(red.item())
            e2e_line["_conv"], h2d_all, d2h_all = (float(x) for x in tot.tolist())
            e2e_line["h2d_bytes_per_step"], e2e_line["d2h_bytes_per_step"] = int(h2d_all), int(d2h_all)
        e2e_line["value"] = e2e_line["_conv"] / e2e_line["_seconds"]
        e2e_line.pop("_conv")
        e2e_line.pop("_seconds")
    # gather tau / reports to rank 0 (north_star: NCCL gather of the results; outside the timed region)
    gather_ms = None
    if world > 1:
        t0 = time.perf_counter()
        for key in ("tau", "rep", "A", "E"):
            x = out[key] if dist.get_backend() == "nccl" else out[key].cpu()
            D.gather_to_root(x, B * world, world, rank)
        torch.cuda.synchronize()
        gather_ms = 1e3 * (time.perf_counter() - t0)
    if rank != 0:
        return
    value = conv_all * args.steps / elapsed
    iters_per_s = inner_all * args.steps / elapsed
    peaks = _peaks()
    kernel_s = float(np.mean(kern_ms)) / 1e3
    achieved = flops / kernel_s / 1e12
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get("k_solve_dram_bytes_per_launch")
    except Exception:
        pass
    binding = None  # the resource ncu shows binding k_solve (shared-memory wavefronts, not the FMA pipe)
    try:
        met = json.load(open(os.path.join(ROOT, "profiles", "r01", "k_solve_s64_full_metrics.json")))
        binding = {"resource": "shared-memory wavefronts (LSU pipe)",
                   "frac": float(met["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"][0]) / 100,
                   "fma_pipe_frac": float(met["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"][0]) / 100,
                   "source": "ncu --set full of k_solve (1184 x 30 iterations), profiles/r01/k_solve_s64_full_metrics.json"}
    except Exception:
        pass
    line = {
        "metric": "rectified patches/s (converged)", "value": value, "unit": "patches/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"config 2: {B} patches 50x50 homography per GPU (tilt_synth seeds [2, idx])",
                   "global_batch": B * world, "per_gpu_batch": B, "patch": f"{m}x{n}", "transform": "homography",
                   "parallelism": f"patch-sharded x{world}", "l2": "flushed between steps (256 MB write)"},
        "inner_iters_per_s": iters_per_s,
        "converged_fraction": conv_all / (B * world),
        "mean_inner_iters_per_patch": inner_all / (B * world),
        "mean_jacobi_sweeps_per_svt": float(np.sum(rep["jacobi_sweeps"]) / max(1, np.sum(rep["inner_iters"]))),
        "roofline": {"bound": "alu", "kernel": "k_solve", "achieved": achieved, "peak": FP32_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic,
                     "peak_note": "FP32 FMA: 148 SMs x 128 lanes x 2 x 1.965 GHz (sm_max_mhz of MEASURED_PEAKS.json); "
                                  "achieved = SURVEY §8(d) model flops from the device counters / event time",
                     "flops_per_launch": flops, "binding": binding},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if gather_ms is not None:
        line["gather_ms"] = gather_ms
    # K1 (warp/Jacobian) standalone HBM roofline over the same batch (first outer iteration's warp)
    if world == 1 and not args.no_k1:
        line["roofline_k1"] = k1_roofline(solver, images, patch_image, boxes, tau0, kind, m, n, p, peaks)
    if e2e_line is not None:
        line["e2e"] = e2e_line
    if world == 1 and args.cpu_sample > 0:
        r = cpu_sample(batch, args.cpu_sample, os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": r["converged"] / r["seconds"], "unit": "patches/s", "cores": r["cores"],
                                "kind": "oracle", "inner_iters_per_s": r["inner_iters"] / r["seconds"],
                                "sample": f"first {r['count']} patches of the same batch, one process per patch"}
    print(json.dumps(line), flush=True)
    solver.close()


def k1_roofline(solver, images, patch_image, boxes, tau0, kind, m, n, p, peaks) -> dict:
    import torch
    B = int(boxes.shape[0])
    reps = 20
    outs = solver.warp(images, patch_image, boxes, tau0, kind)  # warm-up + outputs allocated
    del outs
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dh = torch.empty((B, m, n), dtype=torch.float32, device=images.device)
    J = torch.empty((B, p, m, n), dtype=torch.float32, device=images.device)
    import ctypes
    from paper_1205_5351_b200 import lib
    nrm = torch.empty(B, dtype=torch.float32, device=images.device)
    st = torch.empty(B, dtype=torch.int32, device=images.device)
    n_images, H, W = images.shape

    def launch():
        lib.tilt_warp_batch(solver._h, ctypes.c_void_p(images.data_ptr()), n_images, H, W,
                            ctypes.c_void_p(patch_image.data_ptr()), ctypes.c_void_p(boxes.data_ptr()),
                            ctypes.c_void_p(tau0.data_ptr()), B, kind, m, n, ctypes.c_void_p(dh.data_ptr()),
                            ctypes.c_void_p(J.data_ptr()), ctypes.c_void_p(nrm.data_ptr()),
                            ctypes.c_void_p(st.data_ptr()))
    solver._bind_stream()
    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    # cold-L2 timing: flush (write 256 MB > L2) before every launch, time each launch alone
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=images.device)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0.record()
        launch()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    del flush
    t = float(np.median(ts))
    # algorithmic bytes: distinct source taps (identity tau: (m+1)(n+1) px) + D_hat and J written
    byts = B * 4.0 * ((m + 1) * (n + 1) + m * n * (1 + p))
    achieved = byts / t / 1e9
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get("k_warp_dram_bytes_per_launch")
    except Exception:
        pass
    return {"bound": "hbm", "kernel": "k_warp", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "bytes_per_launch": byts, "us_per_launch": 1e6 * t,
            "note": "standalone K1 over the bench batch at tau0; L2 flushed before each timed launch (median of "
                    f"{reps})"}


def e2e(solver, batch, kind, prm, args) -> dict:
    import torch
    from paper_1205_5351_b200._abi import REPORT_BYTES as T_REPORT_BYTES
    images = np.ascontiguousarray(batch["images"])
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in batch.items()}
    B = batch["boxes"].shape[0]
    p = 8 if kind == 1 else 6
    m, n = int(batch["boxes"][0, 3]), int(batch["boxes"][0, 2])
    solver.solve_host(pinned["images"].numpy(), pinned["patch_image"].numpy(), pinned["boxes"].numpy(),
                      pinned["tau0"].numpy(), kind, prm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    conv = 0
    for _ in range(args.steps):
        r = solver.solve_host(pinned["images"].numpy(), pinned["patch_image"].numpy(), pinned["boxes"].numpy(),
                              pinned["tau0"].numpy(), kind, prm)
        conv += int(np.sum(r["rep"]["status"] == 0))
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    h2d = images.nbytes + batch["patch_image"].nbytes + batch["boxes"].nbytes + B * p * 4
    d2h = B * p * 4 + 2 * B * m * n * 4 + B * T_REPORT_BYTES
    return {"value": conv / t, "unit": "patches/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "tilt_solve_batch_host (host buffers, pinned)", "_conv": conv, "_seconds": t}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=PER_RANK_BATCH)
    ap.add_argument("--cpu-sample", type=int, default=8)
    ap.add_argument("--ref-warmup", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-k1", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: a smoke test of the N > 1 code path on fewer GPUs "
                         "than ranks; never a measurement)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.backend == "gloo":  # smoke test: ranks may share a GPU
            local_rank = local_rank % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
