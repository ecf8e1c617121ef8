"""Multi-process (world size 2, gloo, CPU) checks of the sharding / gather host logic.

No GPU: each rank fabricates per-patch "results" from its patch indices (not the method), gathers
them to rank 0 and rank 0 checks that the reassembled batch equals the single-process one.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import tilt_synth as ts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, out_q):
    import torch.distributed as dist
    from paper_1205_5351_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx = D.shard_indices(total, world, rank)
        # stand-in per-patch results: a deterministic function of the patch's seeded input
        rows = []
        for i in idx:
            p = ts.gen_patch(ts.CONFIGS[1], int(i))
            rows.append([float(i), float(p["canvas"].sum()), float(p["tau_g"][0])])
        x = torch.tensor(np.array(rows, np.float64).reshape(-1, 3))
        g = D.gather_to_root(x, total, world, rank)
        tmax = D.max_over_ranks(float(rank + 1), torch.device("cpu"))
        tsum = D.sum_over_ranks([1.0, float(len(idx))], torch.device("cpu"))
        if rank == 0:
            out_q.put((g.numpy(), tmax, tsum))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 8])
def test_gather_reassembles_batch(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    g, tmax, tsum = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref = []
    for i in range(total):
        p = ts.gen_patch(ts.CONFIGS[1], i)
        ref.append([float(i), float(p["canvas"].sum()), float(p["tau_g"][0])])
    np.testing.assert_array_equal(g, np.array(ref))
    assert tmax == 2.0 and tsum == [2.0, float(total)]


def test_shard_indices_partition():
    from paper_1205_5351_b200 import dist as D
    for total in (0, 1, 5, 1024, 65536):
        for world in (1, 2, 4, 8):
            parts = [D.shard_indices(total, world, r) for r in range(world)]
            allidx = np.sort(np.concatenate(parts)) if total else np.array([])
            np.testing.assert_array_equal(allidx, np.arange(total))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        D.shard_indices(4, 2, 2)


def test_bench_slabs_partition_the_shard():
    """bench.py's step k solves slab k of the rank's shard: the K slabs tile the shard exactly once."""
    import bench
    for total in (1, 7, 8192, 65536):
        for steps in (1, 3, 20):
            sl = bench.slab_bounds(total, steps)
            assert sl[0][0] == 0 and sl[-1][1] == total and len(sl) == steps
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [hi - lo for lo, hi in sl]
            assert max(sizes) - min(sizes) <= 1


def _gpu_worker(rank, world, port, total, out_q):
    import torch.distributed as dist
    import paper_1205_5351_b200 as T
    from paper_1205_5351_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = ts.CONFIGS[2]
        idx = D.shard_indices(total, world, rank)
        b = ts.gen_batch(cfg, 0, total)
        s = T.TiltSolver(0, max_batch=total, max_m=64, max_n=64, max_p=8)
        prm = T.default_params(fixed_outer_iters=2, fixed_inner_iters=15, max_inner=15, max_outer=2)
        out = s.solve(b["images"][idx], np.arange(len(idx), dtype=np.int32), b["boxes"][idx], b["tau0"][idx],
                      cfg.kind, prm)
        got = {k: D.gather_to_root(out[k].cpu(), total, world, rank) for k in ("tau", "A", "E", "rep")}
        if rank == 0:
            ref = s.solve(b["images"], b["patch_image"], b["boxes"], b["tau0"], cfg.kind, prm)
            same = all(torch.equal(got[k], ref[k].cpu()) for k in ("tau", "A", "E", "rep"))
            out_q.put(same)
        s.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gather_of_real_solver_output_is_bit_identical():
    """Two ranks (gloo, sharing one GPU: independent solves, host-side collectives only) solve the
    interleaved shards of 10 config-2 patches; the results gathered on rank 0 equal the single-call
    solve of the whole batch bit for bit (SURVEY §8(c) protocol 4)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    world, total = 2, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    same = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert same
