"""Build tuning variants of libisoquant side by side and time them.

  python tools/variants.py build            # here (CPU): compile every variant
  python tools/variants.py time [--d 128 --bits 3 --dtype f16 --variant full]
                                            # on the GPU box: time each variant

Variants differ only in compile-time knobs (see VARIANTS); the product build is the default one.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {
    "base": [],
    "opsreg": ["-DIQ_OPS_SMEM=0"],          # encoder operators always in registers (8-warp CTAs)
    "nwc12": ["-DIQ_NWC_WIDE=12"],          # 12 compute warps in the wide encoder CTAs
    "nwc20": ["-DIQ_NWC_WIDE=20"],
    "nwc24": ["-DIQ_NWC_WIDE=24"],
    "b3fma": ["-DIQ_B3_ALU=0"],             # b = 3 chain as FSET + FFMA2
    "stage64": ["-DIQ_STAGE_KB=64"],        # 64 KB ring stages
    "stage16": ["-DIQ_STAGE_KB=16"],        # 16 KB ring stages for every encoder
    "dec16kb": ["-DIQ_DEC_STAGE_KB=16"],    # decoder tiles of 16 / 32 KB of output rows at every b
    "dec32kb": ["-DIQ_DEC_STAGE_KB=32"],
    "tchint": ["-DIQ_TC_SPIN=0"],           # suspend-hint waits on tcgen05.commit barriers
    "qjl8": ["-DIQ_QJL_NWC=8"],             # 8 compute warps in the stage-2 kernel
    "attn8": ["-DIQ_ATTN_NWD=8"],           # 8 decoder warps in the attention consumer
    "nopdl": ["-DIQ_PDL=0"],                # no programmatic dependent launch
    "nsplit": ["-DIQ_NORM_SPLIT=1"],        # norm as two interleaved partial sums
    "ring128": ["-DIQ_RING_WIDE_KB=128"],   # smaller TMA ring in the wide encoders
    "ring96": ["-DIQ_RING_WIDE_KB=96"],
    "ring112": ["-DIQ_RING_WIDE_KB=112"],
    "ring160": ["-DIQ_RING_WIDE_KB=160"],
    "stwb": ["-DIQ_STORE_CS=0"],            # ordinary (write-back) output stores
    "dec16": ["-DIQ_TPL_DEC=16"],           # 16 coordinates per lane in the dequantizer
    "dec4": ["-DIQ_TPL_DEC=4"],             # 4 coordinates per lane in the dequantizer
    "grid3": ["-DIQ_GRID_MIN_BITS=3"],      # uniform-grid decision also at b = 3
    "base2": [],                            # second copy of the default (run-order drift)
    "qjl0mma": ["-DIQ_QJL_PASSES=0"],       # timing probe only: no MMAs issued (wrong sketch)
    "qjl1mma": ["-DIQ_QJL_PASSES=1"],       # timing probe only: one MMA pass (inexact sketch)
    "qjlnowait": ["-DIQ_QJL_NOWAIT_PROBE=1"],   # timing probe only: A tile reuse without the MMA wait (racy)
    "norotd": ["-DIQ_QJL_ROTD=0"],          # stage 2 residual in the input domain (2 passes)
    "pu1": ["-DIQ_PAIR_UNROLL=1"],          # one row pair per loop iteration (round-1 form)
    "b3fma64": ["-DIQ_B3_ALU=0", "-DIQ_STAGE_KB=64"],
    "b3fmapu2": ["-DIQ_B3_ALU=0", "-DIQ_PAIR_UNROLL=2"],
    "opsreg12": ["-DIQ_OPS_SMEM=0", "-DIQ_NWC_NARROW=12"],   # operators in registers, 12 compute warps
    "tpl8": ["-DIQ_TPL_K3=8"],              # fused kernel: 8 coordinates per lane (operators in registers)
    "tpl8w12": ["-DIQ_TPL_K3=8", "-DIQ_NWC_WIDE=12"],
    "tpl8w20": ["-DIQ_TPL_K3=8", "-DIQ_NWC_WIDE=20"],
    "qjltc": ["-DIQ_QJL_TCWAIT=1"],
    "qjlrn": ["-DIQ_QJL_MASKSPLIT=0"],
    "qjlhint": ["-DIQ_QJL_MMA_HINT=1"],     # stage-2 MMA warp: parked waits     # stage-2 hi/lo split by RN + convert back (round-1 form)         # stage-2 compute-warp waits without a suspend hint
    "pu2w8": ["-DIQ_PAIR_UNROLL=2", "-DIQ_NWC_WIDE=8"],     # two row pairs per iteration, 8 compute warps
    "pu2w12": ["-DIQ_PAIR_UNROLL=2", "-DIQ_NWC_WIDE=12"],
    "gridpair": ["-DIQ_GRID_PAIR=1"],       # b = 4 grid decision with the rows' FFMAs packed (FFMA2.RM / FFMA2)
    "fhadd": ["-DIQ_FHADD=1"],              # fp16 -> fp32 by FHADD (full-rate) instead of HADD2.F32
    "fhaddb3fma": ["-DIQ_FHADD=1", "-DIQ_B3_ALU=0"],
    "opsreg_r64": ["-DIQ_OPS_SMEM=0", "-DIQ_RING_KB=64"],    # operators in registers, 64 / 128 / 160 KB ring
    "opsreg_r128": ["-DIQ_OPS_SMEM=0", "-DIQ_RING_KB=128"],
    "opsreg_r160": ["-DIQ_OPS_SMEM=0", "-DIQ_RING_KB=160"],
    "opsreg_s16": ["-DIQ_OPS_SMEM=0", "-DIQ_STAGE_KB=16"],   # operators in registers, 16 / 64 KB stages
    "opsreg_s64": ["-DIQ_OPS_SMEM=0", "-DIQ_STAGE_KB=64"],
    "grid5": ["-DIQ_GRID_MIN_BITS=5"],      # b = 4 by the compare chain (no grid decision)
    "wordcodes": ["-DIQ_BYTE_CODES=0"],     # code words gathered by shuffles (round-1/2 form) instead of byte pieces
    "signshf": ["-DIQ_SIGN_SHF=1"],         # code sign bits by funnel shifts
    "k1reg": ["-DIQ_K1_OPS_REG=1"],         # 16-bit quantizer b >= 3: operators in registers, 8 warps
    "k1regshf": ["-DIQ_K1_OPS_REG=1", "-DIQ_SIGN_SHF=1"],
    "tpl8b4": ["-DIQ_TPL_K3B4=8"],          # b = 4 fused kernel: 8 coordinates per lane
    "pu1nwc12": ["-DIQ_PAIR_UNROLL=1", "-DIQ_NWC_NARROW=12"],   # one row pair per iteration, 12 warps
    "attn12": ["-DIQ_ATTN_NWD=12"],         # 12 decoder warps in the attention consumer
    "qjl16": ["-DIQ_QJL_NWC=16"],           # 16 compute warps in the stage-2 kernel
    "stage32": ["-DIQ_STAGE_KB=32"],        # 32 KB ring stages for every encoder
    "ringn128": ["-DIQ_RING_KB=128"],       # 128 KB ring for the 8-warp (register-operator) encoders
    "nwcn6": ["-DIQ_NWC_NARROW=6"],         # 6 compute warps in the register-operator encoders
    "nwcn4": ["-DIQ_NWC_NARROW=4"],
    "b3fmar": ["-DIQ_B3_ALU=0"],            # b = 3 chain as FSET + FFMA2 (register-operator build)
}


def lib_path(name):
    return os.path.join(ROOT, "paper_2603_28430_b200", "build", f"var_{name}", "libisoquant.so")


def build(names, only=None):
    from __graft_entry__ import load_builder
    _build = load_builder()
    for name in names:
        d = os.path.dirname(lib_path(name))
        _build.build(extra=VARIANTS[name], lib=lib_path(name), objdir=d, only=only)
        print("built", name, flush=True)


def time_one(a):
    import torch
    import iqsynth
    import paper_2603_28430_b200 as iq
    tdt = torch.float16 if a.dtype == "f16" else torch.float32
    s = 2 if a.dtype == "f16" else 4
    p = iq.iq_make_params(a.d, a.bits, iq.VARIANTS[a.variant], iqsynth.PARAMS_SEED, device=0)
    from iqsynth import dist as D
    xs, _, _ = D.rank_buffers(2, a.n, a.d, tdt, "cuda", buffers=2)
    ys = [torch.empty_like(x) for x in xs]
    codes = torch.empty((a.n, p.code_bytes), dtype=torch.uint8, device="cuda")
    norms = torch.empty(a.n, dtype=torch.float32, device="cuda")
    iq.iq_quantize(p, xs[0], codes, norms)
    cb = p.code_bytes
    if a.d in (64, 128):
        pq = iq.iq_make_params_qjl(a.d, a.bits, iq.VARIANTS[a.variant], iqsynth.PARAMS_SEED, device=0)
        qj = torch.empty((a.n, a.d // 8), dtype=torch.uint8, device="cuda")
        rn = torch.empty(a.n, dtype=torch.float32, device="cuda")
    out = {}
    for name, fn, bpv in [
        ("rt", lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1]), 2 * a.d * s),
        ("q", lambda i: iq.iq_quantize(p, xs[i & 1], codes, norms), a.d * s + cb + 4),
        ("dq", lambda i: iq.iq_dequantize(p, codes, norms, y=ys[i & 1]), a.d * s + cb + 4),
        ("rte", lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], codes=codes, norms=norms),
         2 * a.d * s + cb + 4),
    ] + ([("qjl", lambda i: iq.iq_quantize_qjl(pq, xs[i & 1], codes, norms, qj, rn), a.d * s + cb + 8 + a.d // 8)]
         if a.d in (64, 128) else []):
        if a.kernels and name not in a.kernels:
            continue
        for i in range(5):
            fn(i)
        torch.cuda.synchronize()
        if a.sustained:                       # the bench protocol: settle under load, then time
            import time as _t
            t0 = _t.time()
            i = 0
            while _t.time() - t0 < a.sustained:
                fn(i)
                i += 1
                if i % 64 == 0:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
        reps = 200 if a.sustained else 40
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        out[name] = (round(us, 1), round(a.n * bpv / us / 1e3 / 6545.0, 3))
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["build", "time", "time1"])
    ap.add_argument("--only", nargs="*", default=list(VARIANTS))
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--variant", default="full")
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--sustained", type=float, default=0.0,
                    help="seconds of untimed settle load before timing (the bench protocol)")
    ap.add_argument("--kernels", nargs="*", default=None, help="subset of rt q dq rte qjl")
    ap.add_argument("--tu", nargs="*", default=None, help="build: only these translation units (basenames)")
    a = ap.parse_args()
    if a.cmd == "build":
        build(a.only, a.tu)
    elif a.cmd == "time1":
        time_one(a)
    else:
        for name in a.only:
            if not os.path.exists(lib_path(name)):
                continue
            env = dict(os.environ, IQ_LIB_PATH=lib_path(name))
            r = subprocess.run([sys.executable, __file__, "time1", "--d", str(a.d), "--bits", str(a.bits),
                                "--dtype", a.dtype, "--variant", a.variant, "--n", str(a.n),
                                "--sustained", str(a.sustained)] + (["--kernels"] + a.kernels if a.kernels else []),
                               env=env, capture_output=True, text=True)
            line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]])[-1]
            print(f"{name:16s} {line}", flush=True)


if __name__ == "__main__":
    main()
