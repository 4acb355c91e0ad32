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


def buffer_seed(config: int, buffer: int) -> int:
    """Base seed of rotating buffer ``buffer`` of config ``config``'s global
    batch (buffer < 1000).  Ranks do not enter the seed: a rank holds rows
    [lo, hi) of the global batch (``weak_shard`` / ``strong_shard``) and
    draws exactly those rows (iqsynth.device_unit_vectors(row0=lo)), whose
    chunk streams are distinct for every (config, buffer, chunk)."""
    assert 0 <= buffer < 1000
    return 1000 * config + buffer


def plan_rows(scaling: str, n: int, world: int, rank: int) -> tuple[int, int, int]:
    """The rows a rank streams: (row0, rows, n_global).  ``weak``: n rows per
    rank, the global batch grows with the world; ``strong``: the global batch
    is n rows, split contiguously (for configs[2]'s [32 layers, 8 heads,
    32768 tokens] cache at G in {1, 2, 4, 8} this is exactly 32/G whole
    layers per rank)."""
    if scaling == "weak":
        lo, hi = weak_shard(n, rank)
        return lo, hi - lo, n * world
    if scaling == "strong":
        lo, hi = strong_shard(n, world, rank)
        return lo, hi - lo, n
    raise ValueError(scaling)


def rank_buffers(config: int, n: int, d: int, torch_dtype, device, scaling: str = "weak",
                 world: int = 1, rank: int = 0, buffers: int = 2):
    """The device-resident input buffers bench.py times for one rank: for each
    rotating buffer j, the rank's rows of config ``config``'s global batch j
    (``plan_rows``), chunk-seeded (``buffer_seed``).  Returns (list of [rows,
    d] tensors, row0, n_global)."""
    import iqsynth
    row0, rows, n_global = plan_rows(scaling, n, world, rank)
    xs = [iqsynth.device_unit_vectors(rows, d, buffer_seed(config, j), torch_dtype, device, row0=row0)
          for j in range(buffers)]
    return xs, row0, n_global


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
