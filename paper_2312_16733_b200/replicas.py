"""Replica plumbing for N GPUs of one node (replicas only).

SubNetAct batches are independent: every GPU holds a full supernet weight
store and serves whole batches, so the data path has no collective.  The
only cross-rank traffic is host-side bookkeeping — which batches a replica
serves and the max-over-ranks device time a throughput number is quoted on —
and it runs over whatever process group the launcher created (NCCL on the
GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def world_rank() -> tuple:
    d = _dist()
    return (d.get_world_size(), d.get_rank()) if d else (1, 0)


def barrier() -> None:
    d = _dist()
    if d and d.get_world_size() > 1:
        d.barrier()


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (e.g. a CUDA-event time) over all ranks."""
    d = _dist()
    if not d or d.get_world_size() == 1:
        return value
    import torch
    dev = (torch.device("cuda", torch.cuda.current_device()) if d.get_backend() == "nccl"
           else torch.device("cpu"))
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


def assign_batches(n_batches: int, world: int, rank: int) -> List[int]:
    """Static weak-scaling shard: batch i is served by replica i % world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_batches, world))


def aggregate_throughput(units_per_rank: Sequence[float], max_seconds: float) -> float:
    """Whole-job units/s: every rank's units over the slowest rank's time."""
    if max_seconds <= 0:
        raise ValueError("non-positive time")
    return float(sum(units_per_rank)) / max_seconds
