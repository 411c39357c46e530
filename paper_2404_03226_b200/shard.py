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


RESULT_KEYS = ("makespan_ms", "worker", "start_ms", "end_ms")


def init_process_group(local: int):
    """One process per GPU over NCCL.  TBSIM_DIST_BACKEND=gloo selects gloo
    (the single-GPU multi-process test runs two ranks on one device, which
    NCCL refuses); returns torch.distributed."""
    import os

    import torch
    import torch.distributed as dist
    backend = os.environ.get("TBSIM_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def allreduce_max(dist, x: float, device) -> float:
    """Max over ranks of a host float (CUDA tensor under NCCL, CPU under gloo)."""
    import torch
    dev = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class AssignmentGather:
    """The north star's final all-gather: every rank's makespans [G] and
    per-task assignments (worker int32, start/end FP64 [T]) onto every GPU,
    in rank order.  Under NCCL the collectives run on the
    device with no host round trip (async_op=True lets a copy stream wait for
    them while the compute stream moves on); under gloo (tests) the tensors
    go through host memory."""

    def __init__(self, dist, local: dict):
        import torch
        self.dist = dist
        self.world = dist.get_world_size()
        self.nccl = dist.get_backend() == "nccl"
        self.out = {k: torch.empty(self.world * local[k].numel(), dtype=local[k].dtype, device=local[k].device)
                    for k in RESULT_KEYS if k in local}

    def __call__(self, local: dict, async_op: bool = False):
        import torch
        if self.nccl:
            works = [self.dist.all_gather_into_tensor(self.out[k], local[k], async_op=async_op) for k in self.out]
            return [w for w in works if w is not None]
        for k in self.out:
            src = local[k].cpu()
            parts = [torch.empty_like(src) for _ in range(self.world)]
            self.dist.all_gather(parts, src)
            self.out[k].copy_(torch.cat(parts))
        return []
