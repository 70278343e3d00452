"""World-size-2 gloo coverage of the multi-GPU host logic (tree sharding and
the statistics reduction that bench.py runs over NCCL on the GPU box)."""

from __future__ import annotations

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_17353_b200.shard import local_trees, reduce_stats, tree_owner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = local_trees(8, rank, world)
    times = torch.tensor([10.0 + rank, 5.0 * (rank + 1)], dtype=torch.float64)
    counts = torch.tensor([len(mine) * 512, rank + 1], dtype=torch.float64)
    t, c = reduce_stats(times, counts, world)
    q.put((rank, mine, t.tolist(), c.tolist()))
    dist.destroy_process_group()


def test_tree_sharding_partitions():
    for world in (1, 2, 4, 8):
        seen = sorted(t for r in range(world) for t in local_trees(8, r, world))
        assert seen == list(range(8))
        assert all(tree_owner(t, world) == t % world for t in range(8))


def test_stats_reduction_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    assert out[0][1] == [0, 2, 4, 6] and out[1][1] == [1, 3, 5, 7]
    for _, _, t, c in out:
        assert t == [11.0, 10.0]          # max over ranks
        assert c == [8 * 512.0, 3.0]      # sum over ranks


def test_bench_spawns_ranks_dry_run():
    """bench.py --gpus 2 re-launches itself under torchrun (two ranks) and runs the per-rank
    host path over gloo: tree-sharded C5 (tree i -> rank i mod 2) and the stats reduction."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "c5",
                        "--dry-run"], capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["ranks_reporting"] == 2
    assert [s["trees"] for s in d["shards"]] == [[0, 2, 4, 6], [1, 3, 5, 7]]
    assert d["rows_total"] == 8 * 512 * 4  # every tree's rows exactly once across the ranks
    assert d["max_times"] == [2.0, 4.0]
