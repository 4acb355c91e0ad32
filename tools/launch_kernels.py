"""Launch one library kernel a few times on device-resident synthetic inputs
(for ncu captures: keep the command short, one GPU).

  python tools/launch_kernels.py --kernel roundtrip --variant full --d 128 --bits 3 --dtype f16
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="roundtrip",
                    choices=["roundtrip", "roundtrip_emit", "quantize", "dequantize", "quantize_qjl", "attention", "all"])
    ap.add_argument("--variant", default="full")
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--no-st2", action="store_true", help="attention: stage 1 only (no sketch term)")
    a = ap.parse_args()
    import torch
    import iqsynth
    import paper_2603_28430_b200 as iq
    tdt = torch.float16 if a.dtype == "f16" else torch.float32
    p = iq.iq_make_params(a.d, a.bits, iq.VARIANTS[a.variant], iqsynth.PARAMS_SEED, device=0)
    x = iqsynth.device_unit_vectors(a.n, a.d, 7, tdt, "cuda")
    y = torch.empty_like(x)
    codes = torch.empty((a.n, p.code_bytes), dtype=torch.uint8, device="cuda")
    norms = torch.empty(a.n, dtype=torch.float32, device="cuda")
    if a.kernel != "roundtrip":           # (the fused kernel needs no codes: keep its launch the only one)
        iq.iq_quantize(p, x, codes, norms)
    if a.kernel in ("quantize_qjl", "attention", "all"):
        pq = iq.iq_make_params_qjl(a.d, a.bits, iq.VARIANTS[a.variant], iqsynth.PARAMS_SEED, device=0)
        qj = torch.empty((a.n, a.d // 8), dtype=torch.uint8, device="cuda")
        rn = torch.empty(a.n, dtype=torch.float32, device="cuda")
    kinds = (["quantize", "dequantize", "roundtrip", "roundtrip_emit", "quantize_qjl", "attention"]
             if a.kernel == "all" else [a.kernel])
    if "attention" in kinds:       # the batch as a cache of 32 heads, 4 queries per head
        H = 32
        nk = a.n // H
        qh = torch.randn((H, 4, a.d), dtype=tdt, device="cuda")
        iq.iq_quantize_qjl(pq, x, codes, norms, qj, rn)
    for k in kinds:
        for _ in range(a.reps):
            if k == "roundtrip":
                iq.iq_roundtrip(p, x, y=y)
            elif k == "roundtrip_emit":
                iq.iq_roundtrip(p, x, y=y, codes=codes, norms=norms)
            elif k == "quantize":
                iq.iq_quantize(p, x, codes, norms)
            elif k == "quantize_qjl":
                iq.iq_quantize_qjl(pq, x, codes, norms, qj, rn)
            elif k == "attention":
                if a.no_st2:
                    iq.iq_attention_scores(pq, codes[:H * nk].view(H, nk, -1), norms[:H * nk].view(H, nk), qh)
                else:
                    iq.iq_attention_scores(pq, codes[:H * nk].view(H, nk, -1), norms[:H * nk].view(H, nk), qh,
                                           qj[:H * nk].view(H, nk, -1), rn[:H * nk].view(H, nk))
            else:
                iq.iq_dequantize(p, codes, norms, y=y)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
