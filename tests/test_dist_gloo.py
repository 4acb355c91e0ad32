"""Multi-process harness logic on CPU with the gloo backend (world_size 2 and
4): row sharding covers the batch exactly once, seeds are disjoint, and the
post-timing statistics combine as MAX (time) / SUM (errors, counts).  The same
code runs over NCCL in bench.py on the GPU box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from iqsynth import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = D.strong_shard(1001, world, rank)
        # a rank-dependent "step time" and per-rank error sums
        ms, se, sx, cnt = D.combine_stats(1.0 + rank, 0.5 * (rank + 1), 2.0, float(hi - lo))
        seeds = [D.shard_seed(2, rank, j) for j in range(2)]
        gathered = [None] * world
        dist.all_gather_object(gathered, (lo, hi, seeds))
        q.put((rank, ms, se, sx, cnt, gathered))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_shards_and_stats(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, se, sx, cnt, gathered in res:
        assert ms == pytest.approx(world)                       # MAX of 1..world
        assert se == pytest.approx(0.5 * world * (world + 1) / 2)
        assert sx == pytest.approx(2.0 * world)
        assert cnt == pytest.approx(1001)                        # shards cover the batch
        spans = sorted((lo, hi) for lo, hi, _ in gathered)
        assert spans[0][0] == 0 and spans[-1][1] == 1001
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        all_seeds = [s for _, _, ss in gathered for s in ss]
        assert len(set(all_seeds)) == len(all_seeds)


def test_single_process_stats_passthrough():
    assert D.combine_stats(3.0, 1.0, 2.0, 5.0) == (3.0, 1.0, 2.0, 5.0)
    assert D.weak_shard(10, 3) == (30, 40)
    sizes = [np.subtract(*D.strong_shard(10, 3, r)[::-1]) for r in range(3)]
    assert sorted(sizes) == [3, 3, 4]
