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
    ap.add_argument("--n", type=int, default=1 << 20, help="vectors per GPU")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernels", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu: headline loop only, no extras")
    return ap.parse_args()


def config_name(a):
    """Which BASELINE.json configs[] entry the arguments describe."""
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
    return {
        "workload": (f"{config_name(a)}: IsoQuant-{a.variant.capitalize()} d={a.d} b={a.bits} "
                     f"{'fp16' if a.dtype == 'f16' else 'fp32'}, {a.n} synthetic unit vectors per GPU"),
        "variant": a.variant, "d": a.d, "bits": a.bits, "io_dtype": a.dtype, "n_per_gpu": a.n,
        "global_vectors": a.n * world, "parallelism": f"dp{world} (vectors sharded by batch)",
        "step": "one fused roundtrip launch (iq_roundtrip) over the batch",
        "l2": "inputs larger than L2 (>=256 MiB per buffer vs 126 MB) and 2 rotating buffer sets "
              "(1 set, or in place, when they do not fit HBM)",
    }


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


# ------------------------------------------------------------------ reference arm
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    if rank != 0:
        return
    import numpy as np
    import iqsynth
    from oracle import iq_oracle as O
    vid = {"full": O.FULL, "fast": O.FAST, "planar2d": O.PLANAR2D}[a.variant]
    po = O.make_params(a.d, a.bits, vid, iqsynth.PARAMS_SEED)
    npdt = np.float16 if a.dtype == "f16" else np.float32
    batch = 8192
    X = iqsynth.unit_vectors(batch, a.d, iqsynth.data_seed(2), npdt)
    for _ in range(a.warmup):
        O.roundtrip(X, po)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        O.roundtrip(X, po)
    t = time.perf_counter() - t0
    v = batch * a.steps / t
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "vectors/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a, world),
        "cpu_baseline": {"value": v, "unit": "vectors/s", "cores": 1, "kind": "oracle",
                         "sample": f"{batch} vectors per step (the paper's batch, P:371) of the same workload, "
                                   f"fp64 NumPy oracle, single process"},
        "e2e": {"value": v, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def cpu_baseline(a, seconds: float):
    """The oracle as it stands, on the host cores, on a bounded sample."""
    import numpy as np
    import iqsynth
    from oracle import iq_oracle as O
    vid = {"full": O.FULL, "fast": O.FAST, "planar2d": O.PLANAR2D}[a.variant]
    po = O.make_params(a.d, a.bits, vid, iqsynth.PARAMS_SEED)
    npdt = np.float16 if a.dtype == "f16" else np.float32
    batch = 8192
    X = iqsynth.unit_vectors(batch, a.d, iqsynth.data_seed(2), npdt)
    O.roundtrip(X[:64], po)
    done, t0 = 0, time.perf_counter()
    while True:
        O.roundtrip(X, po)
        done += batch
        t = time.perf_counter() - t0
        if t >= seconds or done >= 64 * batch:
            break
    return {"value": done / t, "unit": "vectors/s", "cores": 1, "kind": "oracle",
            "sample": f"{done} vectors ({done // batch} batches of {batch}) of the same workload, "
                      f"{t:.1f} s, fp64 NumPy oracle, single process"}


# ------------------------------------------------------------------ our arm
def main():
    a = parse_args()
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist
    import numpy as np

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and rank == 0:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def allreduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=op)
        return t.tolist()

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
    s = 2 if a.dtype == "f16" else 4
    p = iq.iq_make_params(a.d, a.bits, vid, iqsynth.PARAMS_SEED, device=local)
    stream = torch.cuda.current_stream()
    # each rank's shard: its own chunk seeds (weak scaling, no data movement)
    # two rotating buffer sets while they fit; one set (y separate) or in place
    # (y = x, allowed by the ABI) for the largest configs (cfg5: 64 GiB per buffer)
    buf = a.n * a.d * s
    free_b = torch.cuda.mem_get_info(dev)[0]
    nsets = 2 if 4 * buf <= 0.8 * free_b else 1
    inplace = nsets == 1 and 2 * buf > 0.8 * free_b
    xs = [iqsynth.device_unit_vectors(a.n, a.d, D.shard_seed(2, rank, j), tdt, dev)
          for j in range(nsets)]
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
    i = 0
    settle = float(os.environ.get("IQ_SETTLE_S", "0.4"))
    while not a.profile and time.time() - t_load0 < settle:   # untimed clock settle under load
        step(i)
        i += 1
        if i % 64 == 0:
            torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(a.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_end = time.time()
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop(t_load0, t_end) if sampler else None
    # reconstruction sums over every rank's full batch (after timing), then one
    # combine: MAX of the step time, SUM of the statistics (NCCL at N > 1)
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    for j in range(2):
        iq.iq_error_sums(p, xs[j], ys[j], sums)
    ms_max, se_tot, _, cnt_tot = D.combine_stats(ms, *sums.tolist(), 2.0 * a.n * a.d, device=dev)
    mse = None if inplace else se_tot / cnt_tot

    ms_step = ms_max / a.steps
    value = world * a.n / (ms_step / 1e3)
    peak, peak_src = read_peak()
    bpl = a.n * bytes_per_vector("roundtrip", a.d, a.bits, s)
    achieved = bpl / (ms / a.steps / 1e3) / 1e9
    key = f"roundtrip_{a.variant}_d{a.d}_b{a.bits}_{a.dtype}_n{a.n}"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": read_traffic(key),
                "kernel": f"k_encode<{a.dtype},{a.d},{a.bits},{a.variant},roundtrip>",
                "algorithmic_bytes_per_launch": bpl, "peak_source": peak_src}


    out = {
        "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload_config(a, world),
        "hbm_gbs": world * bpl / (ms_step / 1e3) / 1e9,
        "roofline": roofline, "gpu_launches": a.steps, "clocks": clocks,
        "mse": {"value": mse, "closed_form": None, "unit": "per coordinate"},
    }
    if not a.profile:
        try:
            from oracle import iq_oracle as O  # closed form only (no oracle on the path)
            out["mse"]["closed_form"] = O.expected_unit_vector_mse(a.d, a.bits)
        except Exception:
            pass

    # split kernels + fused-with-codes on the headline config (rank-local)
    if not (a.profile or a.no_kernels):
        cb = p.code_bytes
        codes = torch.empty((a.n, cb), dtype=torch.uint8, device=dev)
        norms = torch.empty(a.n, dtype=torch.float32, device=dev)
        kern = {}
        for name, fn in [
            ("quantize", lambda i: iq.iq_quantize(p, xs[i & 1], codes, norms, stream=stream)),
            ("dequantize", lambda i: iq.iq_dequantize(p, codes, norms, y=ys[i & 1], stream=stream)),
            ("roundtrip_emit", lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], codes=codes,
                                                         norms=norms, stream=stream)),
            ("roundtrip", step),
        ]:
            t = time_launches(torch, fn, max(10, a.steps), 3, stream)
            b = a.n * bytes_per_vector(name, a.d, a.bits, s)
            kern[name] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                          "bytes_per_launch": b, "vectors_per_s": a.n / (t / 1e3)}
        if a.d in (64, 128):   # stage-2 residual sketch (tcgen05), NEXT row 1
            pq = iq.iq_make_params_qjl(a.d, a.bits, vid, iqsynth.PARAMS_SEED, device=local)
            qj = torch.empty((a.n, a.d // 8), dtype=torch.uint8, device=dev)
            rn = torch.empty(a.n, dtype=torch.float32, device=dev)
            t = time_launches(torch, lambda i: iq.iq_quantize_qjl(pq, xs[i & 1], codes, norms, qj, rn,
                                                                  stream=stream), max(10, a.steps), 3, stream)
            b = a.n * bytes_per_vector("quantize_qjl", a.d, a.bits, s)
            kern["quantize_qjl"] = {"us": 1e3 * t, "GB/s": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peak,
                                    "bytes_per_launch": b, "vectors_per_s": a.n / (t / 1e3),
                                    "tensor_tflops": a.n * 4 * a.d * a.d / (t / 1e3) / 1e12}
            del qj, rn
        if a.d in (64, 128):   # fused KV-cache decode consumer (NEXT row 2), on this batch as keys
            H = 32                                  # heads of n/32 keys each, 4 queries per head (GQA)
            nk = a.n // H
            qh = torch.randn((H, 4, a.d), dtype=tdt, device=dev)
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
        # context: a plain device-to-device copy of the same bytes (torch's
        # copy kernel, not on our path) timed the same way on this box
        if not inplace:
            t = time_launches(torch, lambda i: ys[i & 1].copy_(xs[i & 1]), max(10, a.steps), 3, stream)
            b = a.n * 2 * a.d * s
            gbs = b / (t / 1e3) / 1e9
            kern["copy_reference"] = {
                "us": 1e3 * t, "GB/s": gbs, "frac": gbs / peak, "bytes_per_launch": b,
                "roundtrip_frac_of_copy": kern["roundtrip"]["GB/s"] / gbs,
                "what": "torch copy_ of x into y (the fused kernel's read + write bytes), library kernel, context only"}
        out["kernels"] = kern
        del codes, norms

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
        t = allreduce([t], dist.ReduceOp.MAX if world > 1 else None)[0]
        out["e2e"] = {"value": world * a.n * a.e2e_steps / t, "unit": "vectors/s",
                      "h2d_bytes_per_step": a.n * a.d * s, "d2h_bytes_per_step": a.n * a.d * s,
                      "timing": "host wall clock around the synchronous iq_host_roundtrip call, max over ranks",
                      "api": "iq_host_roundtrip (pinned host buffers, 2^17-vector chunks, 3 streams)"}
        pl.close()
        del xh, yh

    # the 36-setting grid (18 paper settings x Full/Fast), rank 0 at N=1
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


def sweep(torch, iq, iqsynth, dev, stream, peak):
    n = 1 << 20
    rows = []
    for d in (128, 256, 512):
        base = iqsynth.device_unit_vectors(n, d, iqsynth.data_seed(2, d), torch.float32, dev)
        for dts, tdt, s in (("f16", torch.float16, 2), ("f32", torch.float32, 4)):
            x = base.to(tdt) if tdt != torch.float32 else base
            y = torch.empty_like(x)
            for bits in (2, 3, 4):
                for vname, vid in (("full", 0), ("fast", 1)):
                    p = iq.iq_make_params(d, bits, vid, iqsynth.PARAMS_SEED, device=dev.index)
                    t = time_launches(torch, lambda i: iq.iq_roundtrip(p, x, y=y, stream=stream), 20, 3, stream)
                    b = n * 2 * d * s
                    gbs = b / (t / 1e3) / 1e9
                    rows.append({"variant": vname, "dtype": dts, "d": d, "bits": bits, "us": 1e3 * t,
                                 "GB/s": gbs, "frac": gbs / peak, "vectors_per_s": n / (t / 1e3)})
            del x, y
        del base
        torch.cuda.empty_cache()
    return {"n": n, "kernel": "iq_roundtrip (fused, no code emission)", "rows": rows,
            "min_frac": min(r["frac"] for r in rows)}


if __name__ == "__main__":
    main()
