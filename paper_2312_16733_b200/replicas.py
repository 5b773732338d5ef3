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


# ---------------------------------------------------------------------------
# rank orchestration used by bench.py (and by the gloo test with a stub engine)

def relaunch_under_torchrun(script: str, argv: Sequence[str], gpus: int) -> int:
    """`bench.py --gpus N` under plain python: re-exec the same command as N
    ranks (one process per GPU) with torch.distributed.run on 127.0.0.1.
    Returns the launcher's exit code."""
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           script, *argv]
    return subprocess.call(cmd)


class WallTimer:
    """Host wall-clock timer (stub engines / CPU tests)."""

    def start(self):
        import time
        self.t0 = time.perf_counter()

    def stop(self) -> float:
        import time
        return (time.perf_counter() - self.t0) * 1e3


class CudaTimer:
    """CUDA events on the stream the engine enqueues on; synchronizes."""

    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream

    def start(self):
        self.torch.cuda.synchronize()
        self.e0 = self.torch.cuda.Event(enable_timing=True)
        self.e1 = self.torch.cuda.Event(enable_timing=True)
        self.e0.record(self.stream)

    def stop(self) -> float:
        self.e1.record(self.stream)
        self.torch.cuda.synchronize()
        return self.e0.elapsed_time(self.e1)


def timed_region(step, steps: int, warmup: int, timer, sync=None) -> tuple:
    """W untimed warm-up steps, then exactly `steps` timed ones bracketed by
    a barrier (+ device sync) on both sides.  Returns (this rank's ms, the
    max over ranks)."""
    for i in range(warmup):
        step(i)
    if sync:
        sync()
    barrier()
    timer.start()
    for i in range(steps):
        step(i)
    ms = timer.stop()
    barrier()
    return ms, max_over_ranks(ms)


def load_dispatch_log(path: str) -> List[dict]:
    """tools/_bin/serve_live simulate TSV: the reference router's decisions
    (servesim::run DispatchLog, simcore.hpp:56-70) for N replicas."""
    recs = []
    with open(path) as f:
        for line in f:
            w, sub, cnt, pb, start, pred = line.split()
            recs.append(dict(worker=int(w), subnet=int(sub), count=int(cnt), batch=int(pb),
                             start=int(start), predicted=int(pred)))
    return recs


def rank_dispatches(recs: Sequence[dict], world: int, rank: int) -> List[dict]:
    """Worker w of the N-replica schedule is replica (rank) w: each rank runs
    exactly the dispatches the router sent to its worker, in order."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return [r for r in recs if r["worker"] == rank]


def replay(engine, recs: Sequence[dict], images, id_base: int = 0, stream=None) -> int:
    """Actuate + forward every dispatch (ClampedDispatch: actual_count padded
    to profiled_batch).  Returns the images served."""
    n = 0
    for r in recs:
        engine.actuate(id_base + r["subnet"])
        engine.forward(images, r["count"], r["batch"], None, stream=stream)
        n += r["count"]
    return n
