"""Multi-GPU plumbing: one process per GPU, envs sharded by global index.

Each env's trajectory depends only on (seed, global index, reset count)
(reference bench/runner.py:25-33), so shards need no communication on the
step path; rank r owns the contiguous global range [r*B, (r+1)*B)
(mirroring runner.py:135-143 `_shards`).  The only collectives are the
final reduction of episode statistics and the max-over-ranks time.  Used by
bench.py and examples/ppo_selfplay.py; tests/test_multiproc_gloo.py runs
the same functions with world size 2 on gloo.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

_state = {"backend": None, "device": None}


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment"""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def device(local_rank: int) -> torch.device:
    """this rank's GPU: LOCAL_RANK modulo the visible devices (more ranks
    than GPUs share them round-robin, e.g. a 2-rank gloo run on one GPU)"""
    count = torch.cuda.device_count()
    if count == 0:
        raise RuntimeError("no CUDA device visible to this rank")
    return torch.device("cuda", local_rank % count)


def init(backend: str = "nccl", local_rank: int | None = None) -> None:
    """init_process_group from the torchrun environment (MASTER_ADDR /
    MASTER_PORT / RANK / WORLD_SIZE); NCCL logs its communicator setup
    (NCCL_DEBUG=INFO, subsystem INIT) so the rank count is observable"""
    if backend not in ("nccl", "gloo"):
        raise ValueError(f"bad backend {backend!r}")
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if local_rank is not None and torch.cuda.is_available():
        _state["device"] = device(local_rank)
        torch.cuda.set_device(_state["device"])
    kw = {}
    if backend == "nccl" and _state["device"] is not None:
        kw["device_id"] = _state["device"]
    dist.init_process_group(backend=backend, **kw)
    _state["backend"] = backend


def active() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def backend() -> str | None:
    return _state["backend"] if active() else None


def finish() -> None:
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
    _state["backend"] = None


def barrier() -> None:
    if active():
        if _state["backend"] == "nccl" and _state["device"] is not None:
            dist.barrier(device_ids=[_state["device"].index])
        else:
            dist.barrier()


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


def _all_reduce(t: torch.Tensor, op) -> torch.Tensor:
    """in place; gloo reduces a host copy of a CUDA tensor"""
    if not active():
        return t
    if _state["backend"] == "gloo" and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)
    return t


def reduce_stats(stats: torch.Tensor) -> torch.Tensor:
    """sum (steps, games_completed, illegal) over ranks"""
    return _all_reduce(stats, dist.ReduceOp.SUM)


def max_time(t_ms: float, device) -> float:
    """max over ranks of a device-timed duration"""
    t = torch.tensor([t_ms], dtype=torch.float64, device=device)
    return float(_all_reduce(t, dist.ReduceOp.MAX).item())


def gather_objects(obj) -> list:
    """every rank's `obj`, in rank order (one element without a group)"""
    if not active():
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
