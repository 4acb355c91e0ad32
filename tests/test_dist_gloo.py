"""Multi-process harness logic on CPU with the gloo backend (world_size 2 and
4): the row plans bench.py uses (weak and strong scaling) cover the global
batch exactly once, each rank's generated rows equal the same rows of the
single-process global batch (so the batch and its MSE are identical at every
GPU count), and the post-timing statistics combine as MAX (time) / SUM
(errors, counts).  The same code runs over NCCL in bench.py on the GPU box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import iqsynth
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
        import iqsynth
        lo, rows, n_global = D.plan_rows("strong", 1001, world, rank)
        hi = lo + rows
        # a rank-dependent "step time" and per-rank error sums
        ms, se, sx, cnt = D.combine_stats(1.0 + rank, 0.5 * (rank + 1), 2.0, float(hi - lo))
        # this rank's rows of a chunk-seeded global batch (chunks of 128 rows)
        x = iqsynth.device_unit_vectors(rows, 8, D.buffer_seed(3, 1), torch.float32, "cpu",
                                        chunk_rows=128, row0=lo)
        wlo, wrows, wglobal = D.plan_rows("weak", 300, world, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, (lo, hi, x.numpy(), wlo, wrows, wglobal))
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
        spans = sorted((g[0], g[1]) for g in gathered)
        assert spans[0][0] == 0 and spans[-1][1] == 1001
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        whole = iqsynth.device_unit_vectors(1001, 8, D.buffer_seed(3, 1), torch.float32, "cpu",
                                            chunk_rows=128).numpy()
        for g in gathered:
            assert np.array_equal(g[2], whole[g[0]:g[1]])         # shard == rows of the batch
        weak = sorted((g[3], g[3] + g[4]) for g in gathered)
        assert weak == [(300 * r, 300 * (r + 1)) for r in range(world)]
        assert all(g[5] == 300 * world for g in gathered)


def test_single_process_stats_passthrough():
    assert D.combine_stats(3.0, 1.0, 2.0, 5.0) == (3.0, 1.0, 2.0, 5.0)
    assert D.weak_shard(10, 3) == (30, 40)
    sizes = [np.subtract(*D.strong_shard(10, 3, r)[::-1]) for r in range(3)]
    assert sorted(sizes) == [3, 3, 4]


def test_chunk_streams_are_distinct():
    """no two (buffer, chunk) pairs share a stream (the round-1
    seed + chunk scheme made chunk c of buffer 1 equal chunk c+1 of buffer 0)."""
    a = iqsynth.device_unit_vectors(512, 8, D.buffer_seed(2, 0), torch.float32, "cpu", chunk_rows=128)
    b = iqsynth.device_unit_vectors(512, 8, D.buffer_seed(2, 1), torch.float32, "cpu", chunk_rows=128)
    blocks = [t[i:i + 128].numpy() for t in (a, b) for i in range(0, 512, 128)]
    for i in range(len(blocks)):
        for j in range(i + 1, len(blocks)):
            assert not np.allclose(blocks[i], blocks[j])
    part = iqsynth.device_unit_vectors(200, 8, D.buffer_seed(2, 0), torch.float32, "cpu", chunk_rows=128, row0=100)
    assert torch.equal(part, a[100:300])
