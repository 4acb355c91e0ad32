#!/usr/bin/env python
"""bench.py — IsoQuant stage-1 fused quantize->dequantize on B200.

Workload (BASELINE.json configs[1], headline setting of the north star):
IsoQuant-Full, d=128, 3-bit codes, fp16 storage, 2^20 synthetic unit vectors
per GPU (weak scaling: each rank streams its own shard; no collective on the
hot path).  One STEP = one pass of the whole hot path over one batch: the
fused roundtrip kernel (Algorithm 1 l.1-18) — one launch of
our sm_100a kernel.  The split kernels (quantize = l.1-14 + packing,
dequantize = unpacking + l.15-18) and the fused kernel with code emission are
timed in the same run and reported under "kernels"; the 36-setting grid of
configs[1] (18 paper settings x {Full, Fast}) under "sweep".

Timing: W untimed warm-up steps, a short untimed clock-settle loop, then
EXACTLY K steps bracketed by barrier + cuda.synchronize on both sides, CUDA
events on the launching stream, max over ranks.  Inputs (256 MiB per buffer
at the headline setting) exceed the 126 MB L2 and two buffer sets rotate.
The kernel-level entries ("kernels", "sweep") are the median of three
back-to-back windows of CUDA-event-timed launches.  rank 0 prints ONE JSON
line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

--impl reference times the CPU oracle (oracle/, fp64 NumPy) as the
reference arm on the same config (8192-vector samples per step, the paper's
batch size), on rank 0 only.
"""
from __future__ import annotations

import argparse
import datetime as _dt
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fused quantize-dequantize vectors/s and HBM GB/s vs B200 peak; recon MSE"
FALLBACK_HBM_GBS = 6650.0
VARIANT_NAMES = {0: "full", 1: "fast", 2: "planar2d"}


# BASELINE.json configs as bench presets.  The strong-scaling ones keep the
# global batch (and so its MSE) identical at every GPU count: cfg3's KV cache
# is split by layer (32/G layers per rank), cfg5's 2^26 rows by contiguous
# row ranges.
PRESETS = {
    "headline": dict(variant="full", d=128, bits=3, dtype="f16", n=1 << 20, scaling="weak", config=2,
                     what="configs[1] headline, Full d=128 b=3 fp16, 2^20 vectors per GPU (weak)"),
    "cfg1": dict(variant="full", d=128, bits=3, dtype="f32", n=4096, scaling="weak", config=1,
                 what="configs[0] Full d=128 b=3 fp32, 4096 vectors (L2-resident latency case)"),
    "cfg3": dict(variant="fast", d=128, bits=4, dtype="f16", n=32 * 8 * 32768, scaling="strong", config=3,
                 what="configs[2] KV cache [32 layers, 8 heads, 32768 tokens] Fast d=128 b=4 fp16, "
                      "32/G layers per GPU (strong)"),
    "cfg4": dict(variant="planar2d", d=256, bits=2, dtype="f16", n=1 << 24, scaling="strong", config=4,
                 what="configs[3] 2D d=256 b=2 fp16, 16M vectors (strong)"),
    "cfg5": dict(variant="full", d=512, bits=2, dtype="f16", n=1 << 26, scaling="strong", config=5,
                 what="configs[4] Full d=512 b=2 fp16, 64M vectors across the GPUs (strong)"),
}


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--variant", default="full", choices=["full", "fast", "planar2d"])
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--dtype", default="f16", choices=["f16", "f32"])
    ap.add_argument("--n", "--rows", dest="n", type=int, default=1 << 20,
                    help="vectors per GPU (weak scaling) or in the global batch (strong scaling)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--preset", choices=sorted(PRESETS), default=None,
                    help="a BASELINE.json config: " + "; ".join(f"{k}: {v['what']}" for k, v in PRESETS.items()))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernels", action="store_true")
    ap.add_argument("--no-traffic", action="store_true", help="skip the in-run ncu DRAM-traffic measurement")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu: headline loop only, no extras")
    a = ap.parse_args()
    a.config = 2
    if a.preset:
        for k, v in PRESETS[a.preset].items():
            if k != "what":
                setattr(a, k, v)
    return a


def config_name(a):
    """Which BASELINE.json configs[] entry the arguments describe."""
    if a.preset:
        return PRESETS[a.preset]["what"]
    key = (a.variant, a.d, a.bits, a.dtype)
    if key == ("fast", 128, 4, "f16") and a.n == 32 * 8 * 32768:
        return "configs[2] KV-cache shaped (32 layers x 8 KV heads x 32k tokens)"
    if a.d == 256 and a.bits == 2 and a.dtype == "f16" and a.n == 1 << 24:
        return "configs[3] 16M vectors (2D vs Full/Fast on the same inputs)"
    if key == ("full", 512, 2, "f16") and a.n == 1 << 26:
        return "configs[4] 64M vectors (bandwidth saturation)"
    if a.n == 1 << 20 and key == ("full", 128, 3, "f16"):
        return "configs[1] headline"
    return "configs[1] setting" if a.n == 1 << 20 else "custom"


def workload_config(a, world):
    n_global = a.n * world if a.scaling == "weak" else a.n
    per = "per GPU" if a.scaling == "weak" else "in the global batch"
    return {
        "workload": (f"{config_name(a)}: IsoQuant-{a.variant.capitalize()} d={a.d} b={a.bits} "
                     f"{'fp16' if a.dtype == 'f16' else 'fp32'}, {a.n} synthetic unit vectors {per}"),
        "variant": a.variant, "d": a.d, "bits": a.bits, "io_dtype": a.dtype,
        "n_per_gpu": a.n if a.scaling == "weak" else None, "global_vectors": n_global,
        "parallelism": f"dp{world} (vectors sharded by contiguous row ranges, no collective on the hot path)",
        "step": "one fused roundtrip launch (iq_roundtrip, no code emission) over the rank's rows",
        "data_seeding": "chunk-seeded global batch (iqsynth.dist.rank_buffers): a rank draws exactly its rows",
        "l2": "inputs larger than L2 (>=256 MiB per buffer vs 126 MB) and 2 rotating buffer sets "
              "(1 set, or in place, when they do not fit HBM)" if rank_rows(a, world) * a.d * dsize(a) >= (256 << 20)
              else "L2-resident (a latency configuration, not a bandwidth one)",
    }


def dsize(a) -> int:
    return 2 if a.dtype == "f16" else 4


def rank_rows(a, world) -> int:
    """Rows of the largest rank (the one the max-over-ranks time is set by)."""
    return a.n if a.scaling == "weak" else -(-a.n // world)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampler (100 ms) running across the loaded + timed region."""
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(prefix="iq_clocks_", suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, t0: float, t1: float):
        if self.proc is None:
            return {"error": "nvidia-smi unavailable"}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in open(self.path):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = _dt.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[2]), float(parts[3]), parts[4], parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"error": "no samples"}
        load = [r for r in rows if t0 - 0.05 <= r[0] <= t1 + 0.15] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[4]) if v.lower() == "active"})
        watts = []
        for r in load:
            try:
                watts.append(float(r[3]))
            except ValueError:
                pass
        return {"sm_mhz": statistics.median(r[1] for r in load), "sm_max_mhz": max(r[2] for r in load),
                "reasons": reasons, "samples": len(load),
                "power_w": statistics.median(watts) if watts else None}


# ------------------------------------------------------------------ helpers
def read_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_tensor_peak() -> float:
    """Dense fp16/bf16 tensor peak (TFLOP/s): MEASURED_PEAKS.json's sustained
    cuBLAS bf16 figure (fp16 has the same rate), else the nominal 2250."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d.get("bf16_tflops_sustained") or d["bf16_tflops"])
    except Exception:
        return 2250.0


_UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def parse_ncu_dram(text: str) -> dict:
    """{metric: bytes} for dram__bytes_{read,write}.sum from `ncu --csv` output
    (one launch; non-CSV lines such as the ==PROF== banner are skipped)."""
    import csv
    import io
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    vals = {}
    for row in csv.DictReader(io.StringIO("\n".join(lines))):
        name = row.get("Metric Name")
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = float(row.get("Metric Value", "nan").replace(",", ""))
            vals[name] = v * _UNIT.get(row.get("Metric Unit", "byte"), 1.0)
    return vals


def measure_traffic(a, rows: int, timeout_s: float = 240.0):
    """DRAM bytes (read + write) per launch of the bench's kernel at the bench's
    size, measured in this run: ncu (two counters, one launch after a warm-up
    launch) around tools/launch_kernels.py in a child process.  The child's
    timings are never used.  Returns (bytes or None, note)."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "-k", "regex:k_encode", "--launch-skip", "1", "--launch-count", "1", "--csv", "--print-units", "base",
           sys.executable, os.path.join(ROOT, "tools", "launch_kernels.py"), "--kernel", "roundtrip",
           "--variant", a.variant, "--d", str(a.d), "--bits", str(a.bits), "--dtype", a.dtype,
           "--n", str(rows), "--reps", "2"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
    except Exception as e:  # noqa: BLE001
        return None, f"ncu failed: {type(e).__name__}"
    vals = parse_ncu_dram(r.stdout)
    if len(vals) != 2:
        return None, f"ncu produced no DRAM counters (rc={r.returncode})"
    return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"], (
        "measured in this run: ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch of this kernel "
        "at this size (child process, cold L2)")


def read_traffic(key: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def bytes_per_vector(kind: str, d: int, bits: int, s: int) -> int:
    code = (d * bits + 7) // 8
    return {"roundtrip": 2 * d * s, "roundtrip_emit": 2 * d * s + code + 4,
            "quantize": d * s + code + 4, "dequantize": code + 4 + d * s,
            "quantize_qjl": d * s + code + 4 + d // 8 + 4}[kind]


def time_launches(torch, fn, reps: int, warm: int, stream, repeats: int = 3) -> float:
    """ms per launch: CUDA events on the launching stream, after warm-up;
    the median of `repeats` back-to-back windows of `reps` launches (one
    window can catch a transient clock dip)."""
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    out = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(reps):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps)
    return statistics.median(out)


# ------------------------------------------------------------------ CPU oracle
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _oracle_work(args):
    """One worker: the oracle (as it stands) on `reps` batches of `batch`
    rows of the workload; single-threaded NumPy.  Returns (rows, seconds)."""
    variant, d, bits, dtype, batch, reps, seed = args
    from threadpoolctl import threadpool_limits
    import numpy as np
    import iqsynth
    from oracle import iq_oracle as O
    with threadpool_limits(1):
        po = O.make_params(d, bits, {"full": O.FULL, "fast": O.FAST, "planar2d": O.PLANAR2D}[variant],
                           iqsynth.PARAMS_SEED)
        X = iqsynth.unit_vectors(batch, d, seed, np.float16 if dtype == "f16" else np.float32)
        O.roundtrip(X[:64], po)
        t0 = time.perf_counter()
        for _ in range(reps):
            O.roundtrip(X, po)
        return batch * reps, time.perf_counter() - t0


class OraclePool:
    """The oracle on every host core (one single-threaded process per core,
    spawn start), plus the single-process figure, on bounded samples."""

    def __init__(self, a):
        import multiprocessing as mp
        self.a = a
        self.cores = host_cores()
        self.pool = mp.get_context("spawn").Pool(self.cores)
        self.batch = 8192 if a.d <= 256 else 4096

    def run(self, reps: int):
        """Every core processes `reps` batches; returns (vectors, wall s)."""
        a = self.a
        jobs = [(a.variant, a.d, a.bits, a.dtype, self.batch, reps, iqsynth_seed(a, i)) for i in range(self.cores)]
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_work, jobs)
        return sum(r[0] for r in res), time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def iqsynth_seed(a, i: int) -> int:
    return 1000 * a.config + 500 + i


def cpu_baseline(a, seconds: float):
    """The oracle as it stands, on the host cores, on a bounded sample: one
    process alone, then one process per core (all cores busy)."""
    n1, t1 = _oracle_work((a.variant, a.d, a.bits, a.dtype, 8192 if a.d <= 256 else 4096, 1, 1000 * a.config + 499))
    reps = max(1, int(0.25 * seconds / max(t1, 1e-3)))
    n1, t1 = _oracle_work((a.variant, a.d, a.bits, a.dtype, 8192 if a.d <= 256 else 4096, reps,
                           1000 * a.config + 499))
    pool = OraclePool(a)
    try:
        pool.run(1)                                          # workers up, imports done
        reps_all = max(1, int(0.6 * seconds / max(t1 / reps, 1e-3)))
        nall, tall = pool.run(reps_all)
    finally:
        pool.close()
    return {"value": nall / tall, "unit": "vectors/s", "cores": pool.cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{nall} vectors ({reps_all} batches of {pool.batch} per core on {pool.cores} cores, "
                      f"one single-threaded fp64 NumPy process per core, {tall:.1f} s wall) of the same workload",
            "single_core": {"value": n1 / t1, "unit": "vectors/s", "cores": 1,
                            "sample": f"{n1} vectors, {t1:.1f} s, one process"}}


# ------------------------------------------------------------------ reference arm
def run_reference(a):
    """The CPU oracle as the reference arm, on all host cores, rank 0 only;
    each step = every core coding one bounded batch of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    if rank != 0:
        return
    pool = OraclePool(a)
    try:
        for _ in range(a.warmup):
            pool.run(1)
        done, t = 0, 0.0
        for _ in range(a.steps):
            n, dt = pool.run(1)
            done += n
            t += dt
    finally:
        pool.close()
    v = done / t
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "vectors/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t / a.steps, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a, world),
        "cpu_baseline": {"value": v, "unit": "vectors/s", "cores": pool.cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{pool.batch} vectors per core per step ({pool.cores} cores, one single-threaded "
                                   f"fp64 NumPy oracle process per core) of the same workload"},
        "e2e": {"value": v, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ our arm
def sustained_time(torch, fn, steps: int, stream, settle_s: float, barrier=lambda: None) -> float:
    """ms for `steps` back-to-back launches after an untimed clock-settle loop
    of `settle_s` seconds under the same load (CUDA events on the launching
    stream, synchronize + barrier on both sides)."""
    t0 = time.time()
    i = 0
    while time.time() - t0 < settle_s:
        fn(i)
        i += 1
        if i % 64 == 0:
            torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        fn(i)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    return e0.elapsed_time(e1)


def main():
    a = parse_args()
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and rank == 0:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    # IQ_BENCH_SHARED_GPU=1 (functional check of the N > 1 path on a one-GPU
    # box): every rank on cuda:0, gloo for the statistics (NCCL refuses two
    # ranks on one device).  The throughput is then one GPU's, shared.
    shared = os.environ.get("IQ_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
            one = torch.ones(1)
            dist.all_reduce(one)
            nccl = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                    "allreduce_of_ones": int(one.item()), "shared_gpu": True}
        else:
            # NCCL's init lines (communicator size, transports, NVLS) on stderr,
            # so the communicator is verifiable without mixing into the JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
            one = torch.ones(1, device=dev)
            dist.all_reduce(one)                               # communicator up: counts the ranks
            nccl = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                    "allreduce_of_ones": int(one.item()), "version": ".".join(map(str, torch.cuda.nccl.version()))}

    def barrier():
        if world > 1:
            if shared:
                torch.cuda.synchronize()
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    from __graft_entry__ import load_builder
    _build = load_builder()
    if rank == 0:
        _build.build()
    barrier()
    import iqsynth
    from iqsynth import dist as D
    import paper_2603_28430_b200 as iq

    vid = iq.VARIANTS[a.variant]
    tdt = torch.float16 if a.dtype == "f16" else torch.float32
    s = dsize(a)
    p = iq.iq_make_params(a.d, a.bits, vid, iqsynth.PARAMS_SEED, device=local)
    stream = torch.cuda.current_stream()
    # this rank's rows of the chunk-seeded global batch (weak: its own 2^20
    # rows; strong: its contiguous share, e.g. 32/G layers of the KV cache);
    # two rotating buffer sets while they fit, else one set (y separate) or
    # in place (y = x, allowed by the ABI) for the largest configs
    row0, rows, n_global = D.plan_rows(a.scaling, a.n, world, rank)
    buf = rows * a.d * s
    free_b = torch.cuda.mem_get_info(dev)[0]
    nsets = 2 if 4 * buf <= 0.8 * free_b else 1
    inplace = nsets == 1 and 2 * buf > 0.8 * free_b
    xs, _, _ = D.rank_buffers(a.config, a.n, a.d, tdt, dev, a.scaling, world, rank, buffers=nsets)
    ys = xs if inplace else [torch.empty_like(x) for x in xs]
    if nsets == 1:
        xs, ys = xs * 2, ys * 2

    def step(i):
        iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], stream=stream)

    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(local) if (rank == 0 and not a.profile and not os.environ.get("IQ_NO_SAMPLER")) else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    t_load0 = time.time()
    settle = 0.0 if a.profile else float(os.environ.get("IQ_SETTLE_S", "0.4"))
    ms = sustained_time(torch, step, a.steps, stream, settle, barrier)
    t_end = time.time()
    clocks = sampler.stop(t_load0, t_end) if sampler else None
    # per-rank step times, then one combine: MAX of the step time, SUM of the
    # reconstruction statistics over every rank's rows (NCCL at N > 1)
    per_rank = [ms / a.steps]
    if world > 1:
        g = [None] * world
        dist.all_gather_object(g, ms / a.steps)
        per_rank = g
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    iq.iq_error_sums(p, xs[0], ys[0], sums)
    ms_max, se_tot, _, cnt_tot = D.combine_stats(ms, *sums.tolist(), float(rows * a.d), device=dev)
    mse = None if inplace else se_tot / cnt_tot

    ms_step = ms_max / a.steps
    value = n_global / (ms_step / 1e3)
    peak, peak_src = read_peak()
    bpl = rows * bytes_per_vector("roundtrip", a.d, a.bits, s)
    achieved = bpl / (ms / a.steps / 1e3) / 1e9
    key = f"roundtrip_{a.variant}_d{a.d}_b{a.bits}_{a.dtype}_n{rows}"
    traffic, tsrc = (None, "not measured (--no-traffic / profile mode)")
    if rank == 0 and world == 1 and not (a.profile or a.no_traffic):
        if 2 * rows * a.d * s <= torch.cuda.mem_get_info(dev)[0] // 2:   # the child needs its own x and y
            traffic, tsrc = measure_traffic(a, rows)
        else:
            tsrc = "not measured in this run (the ncu child would not fit next to the bench's buffers)"
    if traffic is None and read_traffic(key) is not None:
        traffic, tsrc = read_traffic(key), tsrc + "; value from profiles/traffic.json (an earlier ncu capture)"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
                "kernel": f"k_encode<{a.dtype},{a.d},{a.bits},{a.variant},MODE 1 (fused, no codes)>",
                "algorithmic_bytes_per_launch": bpl, "peak_source": peak_src,
                "timing": "sustained: 0.4 s untimed settle under load, then the K timed steps (CUDA events)"}

    out = {
        "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload_config(a, world),
        "hbm_gbs": n_global * bytes_per_vector("roundtrip", a.d, a.bits, s) / (ms_step / 1e3) / 1e9,
        "roofline": roofline, "gpu_launches": a.steps, "clocks": clocks,
        "per_rank_ms_per_step": per_rank, "rows_per_rank": [D.plan_rows(a.scaling, a.n, world, r)[1]
                                                            for r in range(world)],
        "mse": {"value": mse, "closed_form": None, "unit": "per coordinate",
                "over": "buffer 0 of every rank's rows (the global batch)"},
    }
    if nccl:
        out["nccl"] = nccl
    if not a.profile:
        try:
            from oracle import iq_oracle as O  # closed form only (no oracle on the path)
            out["mse"]["closed_form"] = O.expected_unit_vector_mse(a.d, a.bits)
        except Exception:
            pass

    # split kernels + fused-with-codes on this config (rank-local)
    if not (a.profile or a.no_kernels):
        out["kernels"] = kernel_entries(torch, iq, iqsynth, a, p, xs, ys, rows, vid, dev, stream, peak, inplace)

    # end to end through the public host-buffer API (H2D + kernel + D2H timed)
    if not (a.profile or a.no_e2e):
        xh = xs[0].cpu().pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        pl = iq.HostPipeline(p, iq.F16 if a.dtype == "f16" else iq.F32, chunk_vectors=1 << 17)
        pl.roundtrip(xh, yh)
        barrier()
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            pl.roundtrip(xh, yh)
        t = time.perf_counter() - t0
        barrier()
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        out["e2e"] = {"value": n_global * a.e2e_steps / t, "unit": "vectors/s",
                      "h2d_bytes_per_step": rows * a.d * s, "d2h_bytes_per_step": rows * a.d * s,
                      "timing": "host wall clock around the synchronous iq_host_roundtrip call, max over ranks",
                      "api": "iq_host_roundtrip (pinned host buffers, 2^17-vector chunks, 3 streams)"}
        pl.close()
        del xh, yh

    # the 36-setting grid (18 paper settings x Full/Fast), rank 0 at N=1,
    # each setting timed like the headline (settle, then rotating buffers)
    if rank == 0 and world == 1 and not (a.profile or a.no_sweep):
        del xs, ys
        torch.cuda.empty_cache()
        out["sweep"] = sweep(torch, iq, iqsynth, dev, stream, peak)

    if rank == 0 and world == 1 and not (a.profile or a.no_cpu):
        out["cpu_baseline"] = cpu_baseline(a, a.cpu_seconds)

    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def kernel_entries(torch, iq, iqsynth, a, p, xs, ys, n, vid, dev, stream, peak, inplace):
    """Every kernel of the path on this config, kernel-level (burst) timing."""
    s = dsize(a)
    cb = p.code_bytes
    codes = torch.empty((n, cb), dtype=torch.uint8, device=dev)
    norms = torch.empty(n, dtype=torch.float32, device=dev)
    kern = {}
    for name, fn in [
        ("quantize", lambda i: iq.iq_quantize(p, xs[i & 1], codes, norms, stream=stream)),
        ("dequantize", lambda i: iq.iq_dequantize(p, codes, norms, y=ys[i & 1], stream=stream)),
        ("roundtrip_emit", lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], codes=codes,
                                                     norms=norms, stream=stream)),
        ("roundtrip", lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], stream=stream)),
    ]:
        t = time_launches(torch, fn, max(10, a.steps), 3, stream)
        b = n * bytes_per_vector(name, a.d, a.bits, s)
        kern[name] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                      "bytes_per_launch": b, "vectors_per_s": n / (t / 1e3)}
    if a.d in (64, 128):   # stage-2 residual sketch (tcgen05), NEXT row 1
        pq = iq.iq_make_params_qjl(a.d, a.bits, vid, iqsynth.PARAMS_SEED, device=dev.index)
        qj = torch.empty((n, a.d // 8), dtype=torch.uint8, device=dev)
        rn = torch.empty(n, dtype=torch.float32, device=dev)
        t = time_launches(torch, lambda i: iq.iq_quantize_qjl(pq, xs[i & 1], codes, norms, qj, rn,
                                                              stream=stream), max(10, a.steps), 3, stream)
        b = n * bytes_per_vector("quantize_qjl", a.d, a.bits, s)
        kern["quantize_qjl"] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                                "bytes_per_launch": b, "vectors_per_s": n / (t / 1e3),
                                "tensor_tflops": n * 4 * a.d * a.d / (t / 1e3) / 1e12}
        del qj, rn
    if n >= 32 * 1024:   # fused KV-cache decode consumer (NEXT row 2), the batch as keys
        H = 32                                  # heads of n/32 keys each, 4 queries per head (GQA)
        nk = n // H
        qh = torch.randn((H, 4, a.d), dtype=xs[0].dtype, device=dev)
        sc = torch.empty((H, 4, nk), dtype=torch.float32, device=dev)
        c3, n3 = codes[:H * nk].view(H, nk, -1), norms[:H * nk].view(H, nk)
        iq.iq_quantize(p, xs[0][:H * nk], codes[:H * nk], norms[:H * nk], stream=stream)
        t = time_launches(torch, lambda i: iq.iq_attention_scores(p, c3, n3, qh, scores=sc, stream=stream),
                          max(10, a.steps), 3, stream)
        b = H * nk * (p.code_bytes + 4 + 4 * 4)
        kern["attention_scores"] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                                    "bytes_per_launch": b, "keys_per_s": H * nk / (t / 1e3),
                                    "shape": f"{H} heads x {nk} keys, 4 queries per head, stage 1"}
        del qh, sc
    # quantize-on-append (NEXT row 2): one decode step of a [32 layers x 8 KV
    # heads] cache (256 slots, one new token each, per-(layer, head) parameter
    # sets), and 64 concurrent sequences (16384 slots) for the bandwidth view
    ps = iq.iq_make_params_sets(a.d, a.bits, vid, iqsynth.PARAMS_SEED, 256, 1, device=dev.index)
    for slots, what in ((256, "one decode step, 32 layers x 8 KV heads"),
                        (16384, "64 sequences x 32 layers x 8 KV heads")):
        if slots > n:
            continue
        cap = 8
        xa = xs[0][:slots]
        ca = torch.empty((slots, cap, ps.code_bytes), dtype=torch.uint8, device=dev)
        na = torch.empty((slots, cap), dtype=torch.float32, device=dev)
        t = time_launches(torch, lambda i: iq.iq_append_kv(ps, xa, ca, na, position=i % cap, stream=stream),
                          max(20, a.steps), 5, stream)
        b = slots * bytes_per_vector("quantize", a.d, a.bits, s)
        kern[f"append_kv_{slots}"] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                                      "keys_per_s": slots / (t / 1e3), "bytes_per_launch": b, "shape": what}
        del ca, na
    # stage 2 at the paper's widths (NEXT row 1): 2^20 rows, b = 3, fp16;
    # d in {256, 512} is the quantizer + the K-chunked sketch kernel.  The
    # tensor roofline counts 4 d m flop per row (hi + lo passes, m = d).
    if a.dtype == "f16" and a.bits == 3 and a.variant == "full" and n >= (1 << 20):
        st2 = {}
        for dd in (128, 256, 512):
            pq = iq.iq_make_params_qjl(dd, 3, vid, iqsynth.PARAMS_SEED, device=dev.index)
            nn = 1 << 20
            xq = iqsynth.device_unit_vectors(nn, dd, 77, torch.float16, dev)
            cq_ = torch.empty((nn, pq.code_bytes), dtype=torch.uint8, device=dev)
            nq_ = torch.empty(nn, dtype=torch.float32, device=dev)
            qj = torch.empty((nn, dd // 8), dtype=torch.uint8, device=dev)
            rn = torch.empty(nn, dtype=torch.float32, device=dev)
            t = time_launches(torch, lambda i: iq.iq_quantize_qjl(pq, xq, cq_, nq_, qj, rn, stream=stream),
                              10, 3, stream)
            b = nn * bytes_per_vector("quantize_qjl", dd, 3, 2)
            fl = nn * 4 * dd * dd
            st2[f"d{dd}"] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                             "tensor_tflops": fl / (t / 1e3) / 1e12,
                             "tensor_frac": fl / (t / 1e3) / 1e12 / read_tensor_peak(),
                             "launches": 1 if dd <= 128 else 2}
            del xq, cq_, nq_, qj, rn
        kern["quantize_qjl_by_width"] = st2
    # context: a plain device-to-device copy of the same bytes (torch's copy
    # kernel, not on our path) timed the same way on this box
    if not inplace:
        t = time_launches(torch, lambda i: ys[i & 1].copy_(xs[i & 1]), max(10, a.steps), 3, stream)
        b = n * 2 * a.d * s
        gbs = b / (t / 1e3) / 1e9
        kern["copy_reference"] = {
            "us": 1e3 * t, "GB/s": gbs, "frac": gbs / peak, "bytes_per_launch": b,
            "roundtrip_frac_of_copy": kern["roundtrip"]["GB/s"] / gbs,
            "what": "torch copy_ of x into y (the fused kernel's read + write bytes), library kernel, context only"}
    return kern


def sweep(torch, iq, iqsynth, dev, stream, peak, steps: int = 20, settle_s: float = 0.3):
    """The 36 settings of configs[1] (d x bits x dtype x {Full, Fast}, 2^20
    rows), each timed like the headline: two rotating buffer sets larger than
    L2, an untimed settle loop under load, then `steps` back-to-back launches
    (CUDA events).  Fractions against the measured HBM peak."""
    from iqsynth import dist as D
    n = 1 << 20
    rows = []
    for d in (128, 256, 512):
        base, _, _ = D.rank_buffers(2, n, d, torch.float32, dev, buffers=2)
        for dts, tdt, s in (("f16", torch.float16, 2), ("f32", torch.float32, 4)):
            xs = [b.to(tdt) if tdt != torch.float32 else b for b in base]
            ys = [torch.empty_like(x) for x in xs]
            for bits in (2, 3, 4):
                for vname, vid in (("full", 0), ("fast", 1)):
                    p = iq.iq_make_params(d, bits, vid, iqsynth.PARAMS_SEED, device=dev.index)
                    fn = lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], stream=stream)
                    for i in range(3):
                        fn(i)
                    # the settle, then the median of three back-to-back
                    # windows (one window can catch a transient clock dip)
                    ws = [sustained_time(torch, fn, steps, stream, settle_s if w == 0 else 0.0) / steps
                          for w in range(3)]
                    t = statistics.median(ws)
                    b = n * 2 * d * s
                    gbs = b / (t / 1e3) / 1e9
                    rows.append({"variant": vname, "dtype": dts, "d": d, "bits": bits, "us": 1e3 * t,
                                 "GB/s": gbs, "frac": gbs / peak, "vectors_per_s": n / (t / 1e3)})
            del xs, ys
        del base
        torch.cuda.empty_cache()
    fp16 = [r["frac"] for r in rows if r["dtype"] == "f16"]
    return {"n": n, "kernel": "iq_roundtrip (fused, no code emission)", "rows": rows,
            "timing": f"sustained: {settle_s} s untimed settle, then the median of three back-to-back windows "
                      f"of {steps} timed launches over 2 rotating buffer sets (CUDA events), per setting",
            "min_frac": min(r["frac"] for r in rows), "min_frac_fp16": min(fp16)}


if __name__ == "__main__":
    main()
