"""Multi-GPU plumbing: patches are independent, so the batch is sharded by patch
across ranks (one process per GPU, torch.distributed); there is no data-path collective. After the
solve, the per-patch results (tau, reports, optionally A/E) are gathered to rank 0 (NCCL on GPUs,
gloo in the CPU tests). Host-side logic only; the solve itself is ``TiltSolver.solve`` per rank.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_indices(total: int, world: int, rank: int) -> np.ndarray:
    """Patch i goes to rank i mod world (interleaved, so heavy and light patches mix)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return np.arange(rank, total, world, dtype=np.int64)


def shard_sizes(total: int, world: int) -> list:
    return [len(range(r, total, world)) for r in range(world)]


def gather_to_root(x: torch.Tensor, total: int, world: int, rank: int, group=None) -> torch.Tensor | None:
    """Gather the per-rank rows of ``x`` (rank r holds patches r, r+world, ...) into patch order on
    rank 0. Ranks with fewer rows are padded for the collective. Returns None on ranks != 0."""
    sizes = shard_sizes(total, world)
    cap = max(sizes)
    pad = torch.zeros((cap,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    out = torch.empty((total,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    for r in range(world):
        out[r::world] = bufs[r][: sizes[r]]
    return out


def max_over_ranks(value: float, device) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values, device) -> list:
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]
