"""Multi-process harness helpers (no method arithmetic): how rows are sharded
across ranks and how the per-rank statistics are combined after timing.

The IsoQuant path partitions by rows (every row is independent, PAPER.md:
Algorithm 1 acts per vector) and the parameters are regenerated from the seed
on every rank, so the hot path needs no collective.  After timing, ranks
combine: the step time (MAX — the job is as slow as its slowest rank), the
reconstruction sums and the row counts (SUM).  These helpers work with any
torch.distributed backend (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def weak_shard(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns global rows [r*n, (r+1)*n)."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def strong_shard(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """Strong scaling: contiguous split of n_global rows, remainder to the
    first ranks (sizes differ by at most one row)."""
    base, rem = divmod(n_global, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def shard_seed(config: int, rank: int, buffer: int) -> int:
    """Data seed of a rank's buffer: disjoint across ranks and buffers."""
    return 1000 * config + 100 * rank + buffer


def combine_stats(step_ms: float, sq_err: float, sq_x: float, count: float, device=None):
    """All-reduce the per-rank statistics: returns (max step ms, total
    squared error, total squared norm, total coordinates).  Call after the
    timed region on every rank."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([step_ms], dtype=torch.float64, device=device)
    s = torch.tensor([sq_err, sq_x, count], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return float(t[0]), float(s[0]), float(s[1]), float(s[2])
