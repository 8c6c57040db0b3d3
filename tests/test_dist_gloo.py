"""Multi-process (world_size 2, gloo, CPU) tests of the benchmark's distributed
plumbing: contiguous b*h sharding covers every unit exactly once, the timing
MAX all-reduce returns the slowest rank, and the reference arm prints only on
rank 0.  The attention path itself has no collective."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = bench.max_over_ranks(float(10 + rank * 5), world)
        bench.barrier(world)
        shards = [bench.shard_units(160, r, world) for r in range(world)]
        q.put((rank, m, bench.shard_units(160, rank, world), shards))
    finally:
        dist.destroy_process_group()


def test_gloo_max_and_shards():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, mine, shards in res:
        assert m == 15.0                    # max over ranks, seen by every rank
        assert mine == shards[rank]


@pytest.mark.parametrize("units,world", [(160, 1), (160, 2), (160, 8), (16, 8), (17, 4), (3, 8), (32, 3)])
def test_shard_units_partition(units, world):
    covered = []
    prev_end = 0
    for r in range(world):
        a, b = bench.shard_units(units, r, world)
        assert a == prev_end and b >= a
        assert b - a in (units // world, units // world + 1)
        covered.extend(range(a, b))
        prev_end = b
    assert covered == list(range(units))


def test_reference_arm_nonzero_rank_is_silent(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class A:
        seqlen, head_dim, causal, warmup, steps, batch, heads = 128, 64, 0, 0, 1, 1, 1
    assert bench.run_reference(A()) is None
