"""Multi-GPU plumbing for the replica layout.

The path does not shard: the reference has one index per process and
`north_star` rules out sharding. With N GPUs each rank holds a full replica
and serves its own query batch (weak scaling); the only collectives are the
broadcast of the trained centroids (so every replica encodes identically) and
the max-over-ranks of device-measured times. Written against a
torch.distributed process group so the same code runs on NCCL (GPU) and gloo
(CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    """(rank, world_size); (0, 1) without an initialised process group."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def share_centroids(cent: np.ndarray | None, shape: tuple[int, int], device) -> np.ndarray:
    """Rank 0's (L, d) f32 centroids on every rank."""
    rank, n = world()
    t = (torch.from_numpy(np.ascontiguousarray(cent, np.float32)).to(device) if rank == 0
         else torch.empty(shape, dtype=torch.float32, device=device))
    if n > 1:
        dist.broadcast(t, 0)
    return t.cpu().numpy()


def max_over_ranks(x: float, device) -> float:
    """The largest of every rank's value (timings: the job is as slow as its slowest rank)."""
    _, n = world()
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if n > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: int, ms_max: float) -> float:
    """Whole-job units/s: every rank's units over the slowest rank's time."""
    _, n = world()
    return units_per_rank * n / (ms_max / 1000.0)
