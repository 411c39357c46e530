"""Multi-GPU plumbing: DAG batches shard by seed range across ranks (one
process per GPU, no traffic during compute); the only collective is the
final all-gather of per-DAG makespans and per-task assignments
(SURVEY.md §8(e)).  Backend-agnostic (NCCL on B200s, gloo in CPU tests)."""
from __future__ import annotations

import numpy as np


def shard_seeds(rank: int, world: int, per_rank: int, base: int = 0) -> np.ndarray:
    """Weak scaling: rank r owns seeds [base + r*per_rank, base + (r+1)*per_rank)."""
    lo = base + rank * per_rank
    return np.arange(lo, lo + per_rank, dtype=np.uint64)


def split_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Strong scaling: contiguous, balanced share of n items."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def all_gather_results(dist, makespans, workers):
    """All-gather equal-sized per-rank result tensors; returns (all_makespans,
    all_workers) concatenated in rank order."""
    import torch
    world = dist.get_world_size()
    ms_out = torch.empty(world * makespans.numel(), dtype=makespans.dtype, device=makespans.device)
    w_out = torch.empty(world * workers.numel(), dtype=workers.dtype, device=workers.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(ms_out, makespans)
        dist.all_gather_into_tensor(w_out, workers)
    else:
        dist.all_gather(list(ms_out.chunk(world)), makespans)
        dist.all_gather(list(w_out.chunk(world)), workers)
    return ms_out, w_out
