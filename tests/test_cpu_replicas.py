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


class StubEngine:
    """Host stand-in for ssn.Engine: records actuations / forwards and sleeps
    in proportion to the dispatched batch (bench.py's rank orchestration
    without a GPU)."""

    def __init__(self):
        self.calls = []
        self.active = None

    def actuate(self, sid):
        self.active = sid

    def forward(self, images, count, profiled_batch, logits, stream=None):
        import time
        assert count <= profiled_batch
        self.calls.append((self.active, count, profiled_batch))
        time.sleep(1e-5 * profiled_batch)


def _replay_rank(rank, world, port, log_path, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        recs = replicas.rank_dispatches(replicas.load_dispatch_log(log_path), world, rank)
        eng = StubEngine()
        served = {}

        def step(_i):
            served["n"] = replicas.replay(eng, recs, None, id_base=3)

        mine, slowest = replicas.timed_region(step, 1, 1, replicas.WallTimer())
        counts = [None] * world
        dist.all_gather_object(counts, served["n"])
        q.put((rank, eng.calls, mine, slowest, counts))
    finally:
        dist.destroy_process_group()


def test_two_rank_slackfit_replay_with_stub_engine(tmp_path):
    """Config-4 orchestration of bench.py on 2 gloo ranks: worker w of the
    router's N-replica dispatch log is replayed by rank w, each dispatch as
    actuate(id_base + subnet) + forward(actual_count, profiled_batch), and
    the whole-job rate is every rank's images over the slowest rank's time."""
    log = tmp_path / "dispatch.tsv"
    rows = [(0, 5, 3, 4, 10, 600), (1, 2, 1, 1, 20, 300), (0, 4, 8, 8, 700, 900),
            (1, 5, 64, 64, 800, 2000), (0, 0, 2, 2, 1700, 310)]
    log.write_text("".join("\t".join(map(str, r)) + "\n" for r in rows))
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_replay_rank, args=(r, world, port, str(log), q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, calls0, ms0, slow0, counts), (_, calls1, ms1, slow1, _) = out
    # each worker's dispatches, in order, with catalog ids offset by id_base
    assert calls0 == [(8, 3, 4), (7, 8, 8), (3, 2, 2)] * 2  # warm-up + timed pass
    assert calls1 == [(5, 1, 1), (8, 64, 64)] * 2
    assert slow0 == slow1 == max(ms0, ms1)
    assert sum(counts) == 3 + 8 + 2 + 1 + 64
    assert replicas.aggregate_throughput(counts, slow0 / 1e3) == pytest.approx(
        78 / (slow0 / 1e3))


def test_bench_gpus_flag_relaunches_ranks():
    """`bench.py --gpus 2` under plain python runs as 2 ranks (torchrun on
    127.0.0.1); the reference arm needs no GPU: rank 0 prints n_gpus 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--image", "32"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(s) for s in out.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
