#!/usr/bin/env python
"""Benchmark of the batched TILT hot path (BASELINE.json metric: rectified patches/s (converged),
LADMAP inner iterations/s, % of FP32 / HBM roofline).

Workload: BASELINE.json configs[4] = config 5, 65 536 patches 50x50 homography (config 2's recipe,
seeded synthetic data from tilt_synth, seeds [5, idx]), the largest configuration that fits one GPU.
The timed region of K steps solves the whole 65 536-patch set exactly once (strong scaling: the set
is fixed, N GPUs split it): rank r owns patches r, r+N, ... (interleaved shards);
step k is one call of the hot entry ``tilt_solve_batch`` on the k-th slab of 65 536 / (N K) of the
rank's patches -- Algorithm 1 for every patch of the slab (warp/Jacobian -> orthonormalise -> LADMAP
inner loop with warm Jacobi SVT -> dtau) until each patch retires. Consecutive slabs alternate
between two handles on two CUDA streams, so a slab's tail (its slowest patches) overlaps the next
slab's start; the whole pass then behaves like one 65 536-patch launch. For N > 1 the per-patch
results (tau, reports, A, E) are gathered to rank 0 over NCCL inside the timed region, which ends
when rank 0 holds them (time = max over ranks).

Prints one JSON line on rank 0. ``--impl reference`` times the fp64 oracle (oracle/) instead, on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import multiprocessing as mp
import os
import platform
import subprocess
import sys
import tempfile
import threading
import time

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")  # the oracle baseline runs one process per patch

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import tilt_synth as ts  # noqa: E402
from tilt_synth import metrics as TM  # noqa: E402

CFG_ID = 5
GLOBAL_BATCH = ts.CONFIGS[CFG_ID].batch  # 65 536
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 148 SMs x 128 FP32 lanes x FMA x sm_max_mhz
METRIC = "rectified patches/s (converged)"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _gen_one(args):
    cfg_id, idx = args
    return ts.gen_patch(ts.CONFIGS[cfg_id], idx)


def gen_shard(cfg_id: int, indices, workers: int = 0) -> dict:
    """Patches ``indices`` of config ``cfg_id`` (one canvas each), generated on the host cores."""
    workers = workers or min(32, os.cpu_count() or 1)
    jobs = [(cfg_id, int(i)) for i in indices]
    count = len(jobs)
    if workers > 1 and count > 8:
        with mp.get_context("fork").Pool(workers) as pool:
            pats = pool.map(_gen_one, jobs, chunksize=64)
    else:
        pats = [_gen_one(j) for j in jobs]
    return {
        "images": np.stack([p["canvas"] for p in pats]),
        "boxes": np.stack([p["box"] for p in pats]),
        "tau0": np.stack([p["tau0"] for p in pats]).astype(np.float32),
        "tau_g": np.stack([p["tau_g"] for p in pats]),
    }


def flops_model(rep, m, n, p, ns_period: int = 4) -> float:
    """Algorithmic FLOPs (SURVEY.md §8(d) model) from the device counters: per LADMAP iteration
    8pmn + 20mn + 4mn^2 + 4n^3/ns_period (the Newton-Schulz step on V after every ns_period-th SVT),
    per Jacobi sweep n(n-1)/2 (12m + 6n) -- every pair of every sweep credited with a rotation."""
    it = float(np.sum(rep["inner_iters"], dtype=np.float64))
    sw = float(np.sum(rep["jacobi_sweeps"], dtype=np.float64))
    return it * (8 * p * m * n + 20 * m * n + 4 * m * n * n + 4 * n ** 3 / max(1, ns_period)) + \
        sw * n * (n - 1) / 2 * (12 * m + 6 * n)


def flops_rotations(rep, m, n, p, ns_period: int = 4) -> float:
    """The same with the Jacobi term from the rotations actually applied (device counter
    ``jacobi_rotations``): every visited pair costs its three column dots (6m), every applied
    rotation its B and V column updates (6m + 6n); a pair below the tolerance costs the dots only."""
    it = float(np.sum(rep["inner_iters"], dtype=np.float64))
    sw = float(np.sum(rep["jacobi_sweeps"], dtype=np.float64))
    rot = float(np.sum(rep["jacobi_rotations"], dtype=np.float64))
    return it * (8 * p * m * n + 20 * m * n + 4 * m * n * n + 4 * n ** 3 / max(1, ns_period)) + \
        sw * n * (n - 1) / 2 * 6 * m + rot * (6 * m + 6 * n)


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


# ------------------------------------------------------------------------------------------------
# the fp64 oracle on the host cores (the cpu_baseline leg and the reference arm)
# ------------------------------------------------------------------------------------------------
def _oracle_job(args):
    import oracle as O
    image, box, tau0 = args
    return O.tilt(image, box, tau0, ts.HOMOGRAPHY)


def cpu_sample(batch: dict, count: int, procs: int) -> dict:
    """The fp64 oracle as it stands on the first ``count`` patches of ``batch``, ``procs`` processes
    (one patch per process at a time, one BLAS thread each)."""
    jobs = [(batch["images"][k], batch["boxes"][k], batch["tau0"][k].astype(np.float64)) for k in range(count)]
    t0 = time.perf_counter()
    if procs > 1:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_job, jobs, chunksize=1)
    else:
        res = [_oracle_job(j) for j in jobs]
    dt = time.perf_counter() - t0
    conv = sum(1 for r in res if r["status"] == 0)
    inner = sum(r["inner_iters"] for r in res)
    return {"seconds": dt, "converged": conv, "inner_iters": inner, "procs": procs, "count": count,
            "patches_per_s": count / dt}


def cpp_sample(batch: dict, count: int, threads: int) -> dict:
    """The C++17 fp64 oracle twin (oracle/tilt_oracle.cpp: its own Jacobi SVD, OpenMP
    over patches) on the first ``count`` patches of ``batch`` with ``threads`` OpenMP threads."""
    from oracle import cpp
    imgs = np.ascontiguousarray(batch["images"][:count], dtype=np.float64)
    t0 = time.perf_counter()
    _, _, _, reps = cpp.solve_batch(imgs, np.arange(count, dtype=np.int32), batch["boxes"][:count],
                                    batch["tau0"][:count].astype(np.float64), ts.HOMOGRAPHY, n_threads=threads)
    dt = time.perf_counter() - t0
    conv = sum(1 for r in reps if r["status"] == 0)
    inner = sum(r["inner_iters"] for r in reps)
    return {"seconds": dt, "converged": conv, "inner_iters": inner, "threads": threads, "count": count,
            "patches_per_s": count / dt}


def cpu_baseline(batch: dict, cores: int) -> dict:
    """the C++ oracle on all host cores (one patch per core) and on one thread (one
    patch), first patches of the bench workload; CPU model read at run time. For context, the numpy
    oracle (LAPACK SVD, one process per patch) on the same all-core sample."""
    allc = cpp_sample(batch, cores, cores)
    one = cpp_sample(batch, 1, 1)
    npy = cpu_sample(batch, cores, cores)
    return {"value": allc["converged"] / allc["seconds"], "unit": "patches/s", "cores": cores, "kind": "oracle",
            "impl": "C++17 fp64 oracle twin (oracle/tilt_oracle.cpp, own Jacobi SVD, OpenMP over patches, "
                    "-O3 -march=x86-64-v3)",
            "cpu_model": cpu_model(), "inner_iters_per_s": allc["inner_iters"] / allc["seconds"],
            "all_patches_per_s": allc["patches_per_s"],
            "sample": f"first {cores} patches of config 5 ({cores} OpenMP threads, {allc['seconds']:.1f} s)",
            "one_thread": {"patches_per_s": one["patches_per_s"],
                           "converged_per_s": one["converged"] / one["seconds"],
                           "inner_iters_per_s": one["inner_iters"] / one["seconds"],
                           "sample": f"first patch, 1 thread ({one['seconds']:.1f} s)"},
            "numpy_oracle": {"converged_per_s": npy["converged"] / npy["seconds"],
                             "inner_iters_per_s": npy["inner_iters"] / npy["seconds"],
                             "sample": f"the same {cores} patches, numpy + LAPACK SVD, one process per patch "
                                       f"({npy['seconds']:.1f} s)"}}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    count = args.cpu_sample or cores
    batch = gen_shard(CFG_ID, range(count))
    vals, inners, secs = [], [], []
    for _ in range(args.warmup if args.ref_warmup else 0):
        cpp_sample(batch, count, min(cores, count))
    for _ in range(args.steps):
        r = cpp_sample(batch, count, min(cores, count))
        vals.append(r["converged"] / r["seconds"])
        inners.append(r["inner_iters"] / r["seconds"])
        secs.append(r["seconds"])
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "patches/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config 5 sample: first {count} of 65536 patches 50x50 homography (C++ fp64 oracle)",
                   "global_batch": count, "patch": "50x50", "transform": "homography"},
        "inner_iters_per_s": float(np.mean(inners)),
        "cpu_baseline": {"value": value, "unit": "patches/s", "cores": min(cores, count), "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "impl": "C++17 fp64 oracle twin (oracle/tilt_oracle.cpp, OpenMP over patches)",
                         "sample": f"first {count} patches of config 5 per step, {min(cores, count)} OpenMP threads"},
        "e2e": {"value": value, "unit": "patches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# the CUDA path
# ------------------------------------------------------------------------------------------------
def slab_bounds(total: int, steps: int) -> list:
    """Step k solves rows [lo_k, hi_k) of the rank's shard: the shard split into ``steps`` slabs."""
    edges = [round(k * total / steps) for k in range(steps + 1)]
    return [(edges[k], edges[k + 1]) for k in range(steps)]


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist
    import paper_1205_5351_b200 as T
    from paper_1205_5351_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = ts.CONFIGS[CFG_ID]
    G = args.global_batch
    m, n, p, kind = cfg.m, cfg.n, cfg.p, cfg.kind
    idx = D.shard_indices(G, world, rank)  # rank r: patches r, r + N, ...
    S = len(idx)
    t_gen = time.perf_counter()
    batch = gen_shard(CFG_ID, idx)
    t_gen = time.perf_counter() - t_gen
    if rank == 0:
        print(f"[bench] generated {S} patches in {t_gen:.1f} s", file=sys.stderr, flush=True)
    slabs = slab_bounds(S, args.steps)
    cap = max(hi - lo for lo, hi in slabs)
    images = torch.as_tensor(batch["images"], device=dev)
    boxes = torch.as_tensor(batch["boxes"], device=dev)
    tau0 = torch.as_tensor(batch["tau0"], device=dev)
    pimg = torch.arange(cap, dtype=torch.int32, device=dev)  # slab-local patch -> image
    nst = max(1, args.streams)
    solvers = [T.TiltSolver(local_rank, max_batch=cap, max_m=m, max_n=n, max_p=p,
                            max_image_elems=cap * 4 * m * n) for _ in range(nst)]
    streams = [torch.cuda.Stream(dev) for _ in range(nst)]
    prm = T.default_params(win_h=m, win_w=n)
    out = {
        "tau": torch.empty((S, p), dtype=torch.float32, device=dev),
        "A": torch.empty((S, m, n), dtype=torch.float32, device=dev),
        "E": torch.empty((S, m, n), dtype=torch.float32, device=dev),
        "rep": torch.empty((S, T.solver._abi.REPORT_BYTES), dtype=torch.uint8, device=dev),
    }

    def step(k: int, slab: int) -> None:
        lo, hi = slabs[slab]
        o = {"tau": out["tau"][lo:hi], "A": out["A"][lo:hi], "E": out["E"][lo:hi], "Y": None,
             "rep": out["rep"][lo:hi]}
        with torch.cuda.stream(streams[k % nst]):
            solvers[k % nst].solve(images[lo:hi], pimg[: hi - lo], boxes[lo:hi], tau0[lo:hi], kind, prm, out=o,
                                   sync=False)

    main = torch.cuda.current_stream(dev)
    for w in range(args.warmup):  # untimed: slabs from the end of the pass
        step(w, (args.steps - 1 - w) % args.steps)
    torch.cuda.synchronize()
    torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev).zero_()  # flush L2 once
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    launches0 = sum(s.launches for s in solvers)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0.record(main)
    for s in streams:
        s.wait_event(t0)
    for k in range(args.steps):
        step(k, k)
    for s in streams:
        main.wait_stream(s)
    gathered = None
    gather_bytes = 0
    if world > 1:  # rank 0 collects every patch's tau / report / A / E (north_star's NCCL gather)
        gathered = {}
        with torch.cuda.nvtx.range("K5 gather tau/reports/A/E to rank 0"):
            for key in ("tau", "rep", "A", "E"):
                x = out[key] if dist.get_backend() == "nccl" else out[key].cpu()
                gathered[key] = D.gather_to_root(x, G, world, rank)
                gather_bytes += int(x.numel() * x.element_size()) * (world - 1)
    t1.record(main)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = sum(s.launches for s in solvers) - launches0
    clk = clocks.stop() if clocks else None
    elapsed = t0.elapsed_time(t1) / 1e3
    if rank == 0:
        print(f"[bench] timed region {elapsed:.2f} s ({args.steps} steps)", file=sys.stderr, flush=True)
    rep = T.reports_to_numpy(out["rep"])
    conv = int(np.sum(rep["status"] == T.CONVERGED))
    inner = int(np.sum(rep["inner_iters"], dtype=np.int64))
    fl_model = flops_model(rep, m, n, p, int(prm.ns_period))
    fl_rot = flops_rotations(rep, m, n, p, int(prm.ns_period))
    stats = [float(conv), float(inner), fl_model, fl_rot, float(launches)]
    if world > 1:
        cdev = dev if dist.get_backend() == "nccl" else "cpu"  # gloo smoke test: host tensors
        tmax = torch.tensor([elapsed], dtype=torch.float64, device=cdev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tot = torch.tensor(stats, dtype=torch.float64, device=cdev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        elapsed = float(tmax.item())
        stats = [float(x) for x in tot.tolist()]
    conv_all, inner_all, fl_model_all, fl_rot_all, launches_all = stats
    # end to end through the host-buffer API (tilt_solve_batch_host), same slabs, same streams
    e2e_line = None
    if not args.no_e2e:
        if world > 1:
            dist.barrier()
        e2e_line = e2e(solvers, batch, slabs, kind, prm, p, m, n)
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
    if rank != 0:
        for s in solvers:
            s.close()
        return
    # results of the whole set on rank 0 (gathered for N > 1)
    if gathered is not None:
        rep_all = T.reports_to_numpy(gathered["rep"])
        tau_all = gathered["tau"].double().cpu().numpy()
        tau_g = np.stack([ts.gen_patch(cfg, int(i))["tau_g"] for i in range(G)]) if args.recovery_all else None
    else:
        rep_all = rep
        tau_all = out["tau"].double().cpu().numpy()
        tau_g = batch["tau_g"]
    value = conv_all / elapsed
    achieved = fl_model_all / elapsed / 1e12
    achieved_rot = fl_rot_all / elapsed / 1e12
    traffic = traffic_note = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get("k_solve_dram_bytes_per_launch")
        traffic_note = prof.get("k_solve_traffic_note")
    except Exception:
        pass
    binding = None
    try:
        met = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))["k_solve_binding"]
        binding = met
    except Exception:
        pass
    status_names = {T.CONVERGED: "converged", T.MAX_OUTER: "max_outer", T.WINDOW_ESCAPE: "window_escape",
                    T.SINGULAR_GRAM: "singular_gram", T.ZERO_PATCH: "zero_patch", T.DIVERGED: "diverged",
                    T.BAD_BOX: "bad_box"}
    stop_names = {0: "none", 1: "objective_change", 2: "dtau", 3: "max_outer"}
    line = {
        "metric": METRIC, "value": value, "unit": "patches/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"config 5: {G} patches 50x50 homography (tilt_synth seeds [5, idx]), "
                               f"one pass per timed region, {args.steps} slabs",
                   "global_batch": G, "per_gpu_batch": S, "slab_patches": cap, "streams": nst,
                   "patch": f"{m}x{n}", "transform": "homography", "parallelism": f"patch-sharded x{world}",
                   "l2": f"not flushed between steps: every step reads its own slab of canvases "
                         f"({cap * 4 * 4 * m * n / 1e6:.0f} MB), the pass reads "
                         f"{S * 4 * 4 * m * n / 1e9:.2f} GB per GPU (L2 126 MB); flushed once before the "
                         f"timed region"},
        "inner_iters_per_s": inner_all / elapsed,
        "converged_fraction": conv_all / G,
        "mean_inner_iters_per_patch": inner_all / G,
        "mean_jacobi_sweeps_per_svt": float(np.sum(rep["jacobi_sweeps"], dtype=np.float64) /
                                            max(1, np.sum(rep["inner_iters"], dtype=np.float64))),
        "status": {status_names.get(int(k), str(k)): int(v) for k, v in
                   zip(*np.unique(rep_all["status"], return_counts=True))},
        "stop_rules": {stop_names.get(int(k), str(k)): int(v) for k, v in
                       zip(*np.unique(rep_all["stop_rule"], return_counts=True))},
        "roofline": {"bound": "alu", "kernel": "k_solve", "achieved": achieved, "peak": FP32_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic,
                     "traffic_note": traffic_note,
                     "peak_note": "FP32 FMA: 148 SMs x 128 lanes x 2 x 1.965 GHz (sm_max_mhz of "
                                  "MEASURED_PEAKS.json; DESIGN.md §4)",
                     "achieved_note": "SURVEY §8(d) model flops from the device counters of all launches / "
                                      "event time of the timed region (k_solve is ~100% of it)",
                     "flops_per_pass": fl_model_all,
                     "rotation_count": {"achieved": achieved_rot, "frac": achieved_rot / FP32_PEAK_TFLOPS,
                                        "flops_per_pass": fl_rot_all,
                                        "note": "Jacobi term from jacobi_rotations: 6m per visited pair + "
                                                "(6m + 6n) per applied rotation"},
                     "binding": binding},
        "gpu_launches": int(launches_all),
        "clocks": clk,
        "gen_seconds": t_gen,
    }
    if tau_g is not None:
        rec = [TM.recovered_p9(tau_all[k], tau_g[k]) for k in range(len(tau_g))]
        err = np.array([TM.table2_error(tau_all[k], tau_g[k]) for k in range(len(tau_g))])
        convm = rep_all["status"][: len(tau_g)] == T.CONVERGED
        line["recovery"] = {
            "rule": "SURVEY P9(ii): H_G^-1 tau* diagonal to 0.02 relative, perspective < 1e-2",
            "patches": len(tau_g), "fraction": float(np.mean(rec)),
            "fraction_of_converged": float(np.mean(np.asarray(rec)[convm])) if convm.any() else None,
            "table2_error_median": float(np.median(err)), "table2_error_mean": float(np.mean(err)),
            "table2_note": "||tau* - tau_G|| / ||tau_G|| (P:1380-1381), normalised coordinates"}
    if world == 1 and not args.no_k1:
        line["recovery_in_basin"] = recovery_in_basin(T, dev)
    if world > 1:
        line["gather"] = {"bytes_to_rank0": gather_bytes, "backend": dist.get_backend(),
                          "note": "tau, reports, A, E of every patch to rank 0, inside the timed region"}
    if world == 1 and not args.no_k1:
        k1n = min(S, args.k1_batch)
        line["roofline_k1"] = k1_roofline(solvers[0], images[:k1n], torch.arange(k1n, dtype=torch.int32, device=dev),
                                          boxes[:k1n], tau0[:k1n], kind, m, n, p, _peaks())
    if e2e_line is not None:
        line["e2e"] = e2e_line
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(batch, args.cpu_sample or (os.cpu_count() or 1))
    print(json.dumps(line), flush=True)
    for s in solvers:
        s.close()


def recovery_in_basin(T, dev, count: int = 256) -> dict:
    """Untimed: free-running solves of SURVEY P9(ii)'s planted-recovery recipe (clean smooth rank-2/3
    textures, 32x32 homography, rotation <= 15 deg, skew <= 0.2, perspective +-1e-3 px; the generator
    of tests/test_gpu_recovery.py, seeds [905, idx]) -- the rectification rate inside TILT's basin,
    beside the config-5 recovery (mostly outside it)."""
    import dataclasses

    import torch
    cfg = dataclasses.replace(ts.CONFIGS[1], corrupt=0.0, config_id=905, rank_lo=2, rank_hi=3,
                              kind=ts.HOMOGRAPHY, persp_px=1e-3)
    pats = [ts.gen_patch(cfg, k, blur_px=1.0) for k in range(count)]
    s = T.TiltSolver(dev.index or 0, max_batch=count, max_m=cfg.m, max_n=cfg.n, max_p=8,
                     max_image_elems=count * 4 * cfg.m * cfg.n)
    out = s.solve(np.stack([q["canvas"] for q in pats]), np.arange(count, dtype=np.int32),
                  np.stack([q["box"] for q in pats]), np.stack([q["tau0"] for q in pats]), cfg.kind,
                  T.default_params(win_h=cfg.m, win_w=cfg.n))
    tau = out["tau"].double().cpu().numpy()
    rep = T.reports_to_numpy(out["rep"])
    s.close()
    ok = [TM.recovered_p9(tau[k], pats[k]["tau_g"]) for k in range(count)]
    return {"recipe": "SURVEY P9(ii): 32x32 homography, clean smooth rank 2-3, theta <= 15 deg, skew <= 0.2",
            "patches": count, "fraction": float(np.mean(ok)),
            "converged_fraction": float(np.mean(rep["status"] == T.CONVERGED)), "timed": False}


def k1_roofline(solver, images, patch_image, boxes, tau0, kind, m, n, p, peaks) -> dict:
    import torch
    from paper_1205_5351_b200 import lib
    B = int(boxes.shape[0])
    reps = 20
    dev = images.device
    dh = torch.empty((B, m, n), dtype=torch.float32, device=dev)
    J = torch.empty((B, p, m, n), dtype=torch.float32, device=dev)
    nrm = torch.empty(B, dtype=torch.float32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    n_images, H, W = images.shape
    images = images.contiguous()

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
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tl = []
    for _ in range(reps):
        flush.zero_()
        e0.record()
        launch()
        e1.record()
        torch.cuda.synchronize()
        tl.append(e0.elapsed_time(e1) / 1e3)
    del flush
    t = float(np.median(tl))
    # algorithmic bytes: distinct source taps (identity tau: (m+1)(n+1) px) + D_hat and J written
    byts = B * 4.0 * ((m + 1) * (n + 1) + m * n * (1 + p))
    achieved = byts / t / 1e9
    peak = float(peaks.get("hbm_gbs", 6536.4))
    traffic = traffic_note = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get("k_warp_dram_bytes_per_launch")
        traffic_note = prof.get("k_warp_traffic_note")
    except Exception:
        pass
    return {"bound": "hbm", "kernel": "k_warp", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note, "bytes_per_launch": byts,
            "us_per_launch": 1e6 * t,
            "patches": B,
            "note": f"standalone K1 over the first {B} patches of the bench workload at tau0; L2 flushed before "
                    f"each timed launch (median of {reps})"}


def e2e(solvers, batch, slabs, kind, prm, p, m, n) -> dict:
    """The same pass through ``tilt_solve_batch_host`` (host buffers in pinned memory; the H2D copy
    of each slab's inputs and the D2H copy of its tau / A / E / reports are inside the timed region).
    Slabs alternate between the handles, one host thread per handle (ctypes drops the GIL)."""
    import torch
    from paper_1205_5351_b200._abi import REPORT_BYTES
    from paper_1205_5351_b200.solver import REPORT_DTYPE
    pin = {k: torch.from_numpy(np.ascontiguousarray(batch[k])).pin_memory().numpy()
           for k in ("images", "boxes", "tau0")}
    S = pin["boxes"].shape[0]
    cap = max(hi - lo for lo, hi in slabs)
    pimg = np.arange(cap, dtype=np.int32)
    tau = torch.empty((S, p), dtype=torch.float32).pin_memory().numpy()
    A = torch.empty((S, m, n), dtype=torch.float32).pin_memory().numpy()
    E = torch.empty((S, m, n), dtype=torch.float32).pin_memory().numpy()
    rep = np.zeros(S, REPORT_DTYPE)
    from paper_1205_5351_b200 import lib
    from paper_1205_5351_b200._abi import check

    def hp(a):
        return a.ctypes.data_as(ctypes.c_void_p)

    streams = [torch.cuda.Stream() for _ in solvers]

    def run(slab_ids, sv, stream):
        with torch.cuda.stream(stream):  # each handle on its own stream: the slabs of the threads overlap
            sv._bind_stream()
        for s in slab_ids:
            lo, hi = slabs[s]
            check(lib.tilt_solve_batch_host(sv._h, hp(pin["images"][lo:hi]), hi - lo, 2 * m, 2 * n, hp(pimg),
                                            hp(pin["boxes"][lo:hi]), hp(pin["tau0"][lo:hi]), hi - lo, kind,
                                            ctypes.byref(prm), hp(tau[lo:hi]), hp(A[lo:hi]), hp(E[lo:hi]),
                                            hp(rep[lo:hi])), "tilt_solve_batch_host")

    nst = len(solvers)
    run([0], solvers[0], streams[0])  # warm-up of the host entry (one slab)
    t0 = time.perf_counter()
    threads = [threading.Thread(target=run, args=(list(range(j, len(slabs), nst)), solvers[j], streams[j]))
               for j in range(nst)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    t = time.perf_counter() - t0
    print(f"[bench] e2e pass {t:.2f} s", file=sys.stderr, flush=True)
    conv = int(np.sum(rep["status"] == 0))
    h2d = pin["images"].nbytes + S * 4 + pin["boxes"].nbytes + pin["tau0"].nbytes
    d2h = S * p * 4 + 2 * S * m * n * 4 + S * REPORT_BYTES
    steps = len(slabs)
    return {"value": conv / t, "unit": "patches/s", "h2d_bytes_per_step": int(h2d / steps),
            "d2h_bytes_per_step": int(d2h / steps),
            "api": f"tilt_solve_batch_host (pinned host buffers), {nst} host threads / handles",
            "timer": "host wall clock around the pass (the entry copies in, solves, copies out, and syncs)",
            "_conv": conv, "_seconds": t}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--global-batch", type=int, default=GLOBAL_BATCH,
                    help="patches of config 5 solved per timed region (default: all 65536)")
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle patches (0: one per host core)")
    ap.add_argument("--k1-batch", type=int, default=GLOBAL_BATCH, help="patches of the standalone K1 launch (default: the whole shard)")
    ap.add_argument("--ref-warmup", action="store_true")
    ap.add_argument("--recovery-all", action="store_true", help="N > 1: regenerate tau_G of every patch on rank 0")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-k1", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
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
