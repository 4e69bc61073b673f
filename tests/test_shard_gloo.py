"""Multi-GPU plumbing on CPU: molecule sharding (no collective on the data
path) and bench.py's barrier / max-over-ranks timing, world_size 2 over gloo."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2211_08506_b200 import shard, synth


def test_plan_shards_cover_and_balance():
    rng = np.random.default_rng(0)
    for world in (1, 2, 4, 8):
        for n in (0, 1, 7, 64, 4096):
            costs = rng.uniform(1, 10, n)
            plan = shard.plan_shards(costs, world)
            assert len(plan) == world
            assert plan[0][0] == 0 and plan[-1][1] == n
            for (a, b), (c, d) in zip(plan, plan[1:]):
                assert b == c and a <= b
            if n >= 64 * world:
                per = [costs[a:b].sum() for a, b in plan]
                assert max(per) - min(per) <= 2 * costs.max()
    with pytest.raises(ValueError):
        shard.plan_shards([1.0], 0)


def test_cost_weighted_shards_for_skewed_config():
    cfg = synth.CONFIGS[4]
    pb = synth.packed_batch(cfg, range(512))
    atoms = np.diff(pb.offsets)
    costs = shard.molecule_costs(atoms, cfg.grid_bytes, bytes_per_atom=20_000.0)
    plan = shard.plan_shards(costs, 8)
    per = [costs[a:b].sum() for a, b in plan]
    assert max(per) / min(per) < 1.05


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench

    dist = bench.Dist(world, rank, rank, backend="gloo")
    dist.barrier()
    # bench.py --scaling strong: every rank plans the same cost-balanced cut
    cfg = synth.CONFIGS[4]
    costs = shard.molecule_costs(synth.atom_counts(cfg, range(100)), cfg.grid_bytes,
                                 shard.BYTES_PER_ATOM)
    rng_ = shard.shard_range(100, rank, world, costs)
    t_max = dist.max(float(rank + 1) * 1.5)
    total = dist.sum(float(len(rng_)))
    dist.close()
    q.put((rank, rng_.start, rng_.stop, t_max, total))


def test_gloo_world2_shards_and_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, m0, s0), (r1, a1, b1, m1, s1) = res
    assert (a0, b1) == (0, 100) and b0 == a1           # disjoint, complete cover
    assert m0 == m1 == 3.0                               # max over ranks
    assert s0 == s1 == 100.0


_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None, timeout=240):
    import subprocess
    import sys

    e = {k: v for k, v in os.environ.items()
         if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(_ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=timeout, env=e, cwd=_ROOT)


def test_bench_gpus2_spawns_two_ranks_dry_run():
    """`bench.py --gpus 2` without a launcher re-executes itself under
    torch.distributed.run with 2 ranks; the strong-scaling cut of cfg1's
    1024 molecules is complete and disjoint (kernels skipped: --dry-run)."""
    import json

    res = _bench("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "1")
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["global_batch"] == 1024 and line["scaling"] == "strong"
    ranks = line["per_rank"]
    assert [r["rank"] for r in ranks] == [0, 1]
    assert ranks[0]["start"] == 0 and ranks[0]["stop"] == ranks[1]["start"]
    assert ranks[1]["stop"] == 1024
    assert sum(r["molecules"] for r in ranks) == 1024


def test_bench_rejects_world_size_mismatch():
    res = _bench("--gpus", "3", "--dry-run", env={"WORLD_SIZE": "2", "RANK": "0"})
    assert res.returncode == 2
    assert "WORLD_SIZE=2" in res.stderr


def _rank_shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS[4]
    counts = synth.atom_counts(cfg, range(300))
    plain = shard.rank_shard(300)
    balanced = shard.rank_shard(300, atom_counts=counts, grid_bytes=cfg.grid_bytes)
    # every rank got a disjoint range; all-gathered they cover the batch
    got = [None] * world
    tdist.all_gather_object(got, (plain.start, plain.stop, balanced.start, balanced.stop))
    tdist.destroy_process_group()
    q.put((rank, shard.rank_world(), got))


def test_rank_shard_under_a_process_group():
    """shard.rank_shard reads rank / world from torch.distributed (the user's
    DDP job): disjoint contiguous ranges covering the
    batch, by count and by estimated cost."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = res[0][2]
    assert got == res[1][2]
    (a0, b0, c0, d0), (a1, b1, c1, d1) = got
    assert (a0, b0, a1, b1) == (0, 150, 150, 300)
    assert c0 == 0 and d0 == c1 and d1 == 300
    assert res[0][1] == (0, 1)        # after destroy_process_group: the environment default


def test_rank_world_from_environment(monkeypatch):
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("WORLD_SIZE", "8")
    assert shard.rank_world() == (3, 8)
    assert shard.rank_shard(80) == range(30, 40)
