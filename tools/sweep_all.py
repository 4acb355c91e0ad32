"""Time the fused roundtrip (and quantize / dequantize) on every GPU
configuration: d in {64, 128, 256, 512} x bits 1-4 x Full/Fast/2D x
fp32/fp16/bf16, 2^20 rows each, CUDA events over 20 back-to-back launches on
two rotating buffer sets (inputs > L2).  Writes one JSON document.

  python tools/sweep_all.py [--out gpurun_out/sweep_all.json] [--n 1048576]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep_all.json")
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--peak", type=float, default=6650.0, help="GB/s (fallback of B200_PROFILING.md)")
    a = ap.parse_args()
    import torch
    import iqsynth
    import paper_2603_28430_b200 as iq

    def timed(fn, reps=20, warm=3):
        for i in range(warm):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3   # us

    rows = []
    n = a.n
    for d in (64, 128, 256, 512):
        base = iqsynth.device_unit_vectors(n, d, 2024 + d, torch.float32, "cuda")
        for dtn, tdt, s in (("f32", torch.float32, 4), ("f16", torch.float16, 2), ("bf16", torch.bfloat16, 2)):
            xs = [base.to(tdt), base.flip(0).to(tdt)]
            ys = [torch.empty_like(xs[0]) for _ in range(2)]
            for bits in (1, 2, 3, 4):
                codes = torch.empty((n, d * bits // 8), dtype=torch.uint8, device="cuda")
                norms = torch.empty(n, dtype=torch.float32, device="cuda")
                for vn, v in (("full", iq.FULL), ("fast", iq.FAST), ("planar2d", iq.PLANAR2D)):
                    p = iq.iq_make_params(d, bits, v, iqsynth.PARAMS_SEED, device=0)
                    t_rt = timed(lambda i: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1]))
                    t_q = timed(lambda i: iq.iq_quantize(p, xs[i & 1], codes, norms))
                    t_dq = timed(lambda i: iq.iq_dequantize(p, codes, norms, y=ys[i & 1]))
                    cb = d * bits // 8 + 4
                    rows.append({
                        "d": d, "dtype": dtn, "bits": bits, "variant": vn,
                        "roundtrip_us": t_rt, "roundtrip_frac": n * 2 * d * s / t_rt / 1e3 / a.peak,
                        "quantize_us": t_q, "quantize_frac": n * (d * s + cb) / t_q / 1e3 / a.peak,
                        "dequantize_us": t_dq, "dequantize_frac": n * (d * s + cb) / t_dq / 1e3 / a.peak})
                del codes, norms
            del xs, ys
        del base
        torch.cuda.empty_cache()
    out = {"n": n, "peak_gbs": a.peak, "peak_source": "fallback (B200_PROFILING.md 6.65 TB/s)",
           "timing": "CUDA events, 20 back-to-back launches after 3 warm-ups, 2 rotating buffer sets", "rows": rows,
           "min_roundtrip_frac": min(r["roundtrip_frac"] for r in rows),
           "min_roundtrip_frac_bits_2_4": min(r["roundtrip_frac"] for r in rows if r["bits"] >= 2)}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("n", "min_roundtrip_frac", "min_roundtrip_frac_bits_2_4")}))


if __name__ == "__main__":
    main()
