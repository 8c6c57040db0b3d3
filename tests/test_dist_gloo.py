"""Multi-process (world_size 2, gloo, CPU) tests of the benchmark's distributed
plumbing: contiguous b*h sharding covers every unit exactly once, rank 0's scatter
and gather reassemble per-unit results in order, the timing MAX all-reduce returns
the slowest rank, `--gpus N` fails loudly without N devices, and the reference arm
prints only on rank 0.  The attention path itself has no collective."""
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


def _stub_unit_op(x):
    """A per-unit computation (each (b,h) unit transformed independently, like the
    attention step): a running sum over rows plus the unit's own mean."""
    return x.cumsum(dim=1) + x.mean(dim=(1, 2), keepdim=True)


def _exchange_worker(rank, world, port, n_units, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, d = 5, 3
        glob = None
        if rank == 0:
            g = torch.Generator().manual_seed(5)
            glob = torch.randn(n_units, N, d, generator=g)
        mine = bench.scatter_units(glob, n_units, (N, d), torch.float32, torch.device("cpu"), rank, world)
        u0, u1 = bench.shard_units(n_units, rank, world)
        res = _stub_unit_op(mine) if mine.shape[0] else mine
        lse_like = res.sum(dim=2)                       # a [U, N] output, like L
        full = bench.gather_units(res, n_units, rank, world)
        full_l = bench.gather_units(lse_like, n_units, rank, world)
        if rank == 0:
            ok = torch.equal(full, _stub_unit_op(glob)) and torch.equal(full_l, _stub_unit_op(glob).sum(dim=2))
            q.put((rank, tuple(mine.shape), (u0, u1), ok))
        else:
            q.put((rank, tuple(mine.shape), (u0, u1), full is None and full_l is None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_units", [5, 4, 1])
def test_gloo_scatter_compute_gather(n_units):
    """rank 0 scatters contiguous (b,h) shards (uneven and empty ones included), each
    rank runs a per-unit stub, rank 0 gathers: the reassembled result equals the
    stub applied to the whole array, unit for unit and in order."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, n_units, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, shape, (u0, u1), ok in res:
        assert ok, rank
        assert shape == (u1 - u0, 5, 3)
    assert res[0][2][0] == 0 and res[-1][2][1] == n_units


def test_bench_gpus_without_devices_fails_loudly():
    """`bench.py --gpus 2` with fewer than 2 CUDA devices must exit non-zero with a
    message instead of silently running one process."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(bench.__file__), "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "needs 2 CUDA devices" in r.stderr
    assert r.stdout.strip() == ""


def test_bench_world_mismatch_fails(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "4")
    with pytest.raises(SystemExit) as e:
        bench.relaunch_if_needed(2)
    assert e.value.code == 2


def test_configs_follow_baseline():
    """--config names map to BASELINE.json configs and SURVEY §8's row sizes."""
    c = {n: bench.resolve_config(bench.parse_args(["--config", n])) for n in bench.CONFIGS}
    assert (c["ps128"]["d"], c["ps128"]["H"], c["ps128"]["N"], c["ps128"]["B"]) == (128, 16, 8192, 2)
    assert c["ps128"]["scaling"] == "weak" and not c["ps128"]["causal"]
    assert (c["gpt"]["H"], c["gpt"]["d"], c["gpt"]["N"], c["gpt"]["B"], c["gpt"]["causal"]) == (20, 128, 8192, 8, True)
    assert c["gpt"]["scaling"] == "strong"
    assert [bench.shard_units(160, r, 8) for r in range(8)][-1] == (140, 160)
    assert (c["lc"]["B"], c["lc"]["H"], c["lc"]["dtype"], c["lc"]["causal"]) == (1, 16, "fp16", True)
    assert (c["ps64"]["d"], c["ps64"]["H"]) == (64, 32)


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

    assert bench.run_reference(bench.parse_args(["--impl", "reference", "--steps", "1"])) is None
