"""Multi-GPU plumbing: one process per GPU, envs sharded by global index.

Each env's trajectory depends only on (seed, global index, reset count)
(reference bench/runner.py:25-33), so shards need no communication on the
step path; rank r owns the contiguous global range [r*B, (r+1)*B)
(mirroring runner.py:135-143 `_shards`).  The only collective is the final
reduction of episode statistics.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment"""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, world_size: int, envs_per_rank: int) -> tuple[int, int]:
    """(index_base, n) of this rank's envs (weak scaling: fixed per rank)"""
    if not 0 <= rank < world_size:
        raise ValueError("rank out of range")
    return rank * envs_per_rank, envs_per_rank


def split(total: int, world_size: int, rank: int) -> tuple[int, int]:
    """(index_base, n) for strong scaling: `total` envs split as evenly as
    runner.py:135-143 does (the first `total % world` ranks get one more)"""
    base, extra = divmod(total, world_size)
    n = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, n


def reduce_stats(stats: torch.Tensor) -> torch.Tensor:
    """sum (steps, games_completed, illegal) over ranks; NCCL on GPUs"""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM)
    return stats


def max_time(t_ms: float, device) -> float:
    """max over ranks of a device-timed duration"""
    t = torch.tensor([t_ms], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
