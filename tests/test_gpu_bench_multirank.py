"""The bench's N > 1 path on hardware: two ranks under torch.distributed.run,
both on cuda:0 (IQ_BENCH_SHARED_GPU=1, gloo for the statistics), strong
scaling over a chunk-seeded global batch.  Checks the JSON contract of the
multi-rank line: the rank count, the per-rank row plan covering the batch
exactly, per-rank times, the max-over-ranks step time, and a global MSE
equal to the closed form."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_strong_scaling_line():
    n = 3 * (1 << 18) + 1000          # a remainder the last rank takes
    # (--rows, not --n: torch.distributed.run would read "--n" as an
    # abbreviation of its own options)
    env = dict(os.environ, IQ_BENCH_SHARED_GPU="1", IQ_NO_SAMPLER="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--rows", str(n), "--scaling", "strong", "--steps", "5", "--warmup", "3",
           "--no-sweep", "--no-cpu", "--no-kernels", "--no-traffic", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["nccl"]["world_size"] == 2 and d["nccl"]["allreduce_of_ones"] == 2
    assert sum(d["rows_per_rank"]) == n and len(d["rows_per_rank"]) == 2
    assert len(d["per_rank_ms_per_step"]) == 2
    assert abs(d["ms_per_step"] - max(d["per_rank_ms_per_step"])) <= 1e-9 * max(d["per_rank_ms_per_step"]) + 1e-12
    assert d["config"]["global_vectors"] == n
    mse, cf = d["mse"]["value"], d["mse"]["closed_form"]
    assert abs(mse - cf) <= 0.02 * cf, (mse, cf)
