"""Time iq_attention_scores on a KV-cache shaped workload (cfg3 layout:
heads = layers x KV heads, n_keys tokens, n_q queries per KV head).

  python tools/attn_bench.py [--heads 256 --keys 32768 --d 128 --bits 4 --variant fast --nq 4]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=256)
    ap.add_argument("--keys", type=int, default=32768)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--variant", default="fast")
    ap.add_argument("--nq", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch, iqsynth
    import paper_2603_28430_b200 as iq
    n = a.heads * a.keys
    st2 = a.d <= 128 or (a.d == 256 and a.bits <= 3)   # the consumer's stage-2 widths
    mk = iq.iq_make_params_qjl if st2 else iq.iq_make_params
    p = mk(a.d, a.bits, iq.VARIANTS[a.variant], iqsynth.PARAMS_SEED, device=0)
    codes = torch.empty((n, p.code_bytes), dtype=torch.uint8, device="cuda")
    norms = torch.empty(n, dtype=torch.float32, device="cuda")
    qj = torch.empty((n, a.d // 8), dtype=torch.uint8, device="cuda")
    rn = torch.empty(n, dtype=torch.float32, device="cuda")
    chunk = 1 << 22
    for r0 in range(0, n, chunk):
        m = min(chunk, n - r0)
        x = iqsynth.device_unit_vectors(m, a.d, 9000 + r0 // chunk, torch.float16, "cuda")
        if st2:
            iq.iq_quantize_qjl(p, x, codes[r0:r0 + m], norms[r0:r0 + m], qj[r0:r0 + m], rn[r0:r0 + m])
        else:
            iq.iq_quantize(p, x, codes[r0:r0 + m], norms[r0:r0 + m])
    del x
    q = torch.randn((a.heads, a.nq, a.d), dtype=torch.float16, device="cuda")
    scores = torch.empty((a.heads, a.nq, a.keys), dtype=torch.float32, device="cuda")
    c3, n3 = codes.view(a.heads, a.keys, -1), norms.view(a.heads, a.keys)
    q3, r3 = qj.view(a.heads, a.keys, -1), rn.view(a.heads, a.keys)
    out = {}
    for name, fn, bpk in [
        ("stage1", lambda: iq.iq_attention_scores(p, c3, n3, q, scores=scores), p.code_bytes + 4 + 4 * a.nq),
        ("stage1+2", lambda: iq.iq_attention_scores(p, c3, n3, q, q3, r3, scores=scores),
         p.code_bytes + 4 + a.d // 8 + 4 + 4 * a.nq),
    ][:2 if st2 else 1]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.reps * 1e3
        out[name] = {"us": round(us, 1), "keys_per_s": n / us * 1e6, "GB/s": n * bpk / us / 1e3,
                     "bytes_per_key": bpk}
    print(json.dumps({"workload": vars(a), **out}))


if __name__ == "__main__":
    main()
