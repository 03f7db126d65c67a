"""Multi-GPU plumbing for the replicas-only path.

RN-AMG setup has global sequential dependencies (greedy aggregation pass 1,
forward Gauss-Seidel) and every Krylov iteration needs global reductions, so
the path does not shard along one exchange step.  With N GPUs each rank runs
its own independent problem (weak scaling); torch.distributed (NCCL on the
GPU box, gloo in the CPU tests) only provides the barrier around the timed
region and the max-over-ranks of the measured times.  No data-path collective.
"""
from __future__ import annotations

import os


def env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str):
    import torch.distributed as dist
    ws, rank, _ = env()
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group(backend, rank=rank, world_size=ws)
    return dist if ws > 1 else None


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(value: float, dist, device=None) -> float:
    """The job's time is the slowest rank's time."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist, device=None) -> float:
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
