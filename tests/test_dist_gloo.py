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
