"""Multi-GPU partitioning of independent trees.

Trees / requests share no cache state: tree i lives on rank ``i % world`` with
its own cache shard, so the data path has no collective.  The only collective
is one reduction of a small statistics vector after a timed interval (NCCL on
the GPU box; gloo in the CPU tests): max of elapsed times, sum of counters.
"""

from __future__ import annotations

import torch


def tree_owner(tree_id: int, world: int) -> int:
    return tree_id % world


def local_trees(n_trees: int, rank: int, world: int) -> list[int]:
    return [t for t in range(n_trees) if tree_owner(t, world) == rank]


def reduce_stats(times: torch.Tensor, counts: torch.Tensor, world: int):
    """(max over ranks of times, sum over ranks of counts); identity at world 1."""
    if world <= 1:
        return times.clone(), counts.clone()
    import torch.distributed as dist

    t = times.clone()
    c = counts.clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return t, c
