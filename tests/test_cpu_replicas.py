"""N > 1 replica path on CPU: two gloo ranks exercise the host-side
plumbing bench.py uses under torchrun (paper_2312_16733_b200/replicas.py):
the max-over-ranks timing reduction, the static batch shard (weak scaling,
no data-path collective) and the whole-job throughput."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2312_16733_b200 import replicas


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assert replicas.world_rank() == (world, rank)
        replicas.barrier()
        ms = 10.0 + 5.0 * rank  # this rank's "device time"
        slowest = replicas.max_over_ranks(ms)
        shard = replicas.assign_batches(11, world, rank)
        shards = [None] * world
        dist.all_gather_object(shards, shard)
        q.put((rank, slowest, shards))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_replicas():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, slowest, shards in out:
        assert slowest == 15.0  # every rank quotes the slowest rank's time
        flat = sorted(b for s in shards for b in s)
        assert flat == list(range(11))  # each batch served exactly once
        assert all(len(set(a) & set(b)) == 0 for i, a in enumerate(shards) for b in shards[i + 1:])


def test_single_process_fallbacks():
    assert replicas.world_rank() == (1, 0)
    assert replicas.max_over_ranks(3.5) == 3.5
    replicas.barrier()
    assert replicas.assign_batches(5, 1, 0) == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        replicas.assign_batches(5, 2, 2)
    # weak scaling: 2 ranks x 192 images over the slowest rank's 4 ms
    assert replicas.aggregate_throughput([192, 192], 0.004) == pytest.approx(96000.0)
    with pytest.raises(ValueError):
        replicas.aggregate_throughput([1], 0.0)
