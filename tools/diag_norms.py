"""Diagnose norm/codes mismatches at large n: compare the library's norms with
torch's row norms for each encoder kernel on device-resident data."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--n", type=int, default=1 << 20)
    a = ap.parse_args()
    import torch
    import iqsynth
    import paper_2603_28430_b200 as iq
    tdt = torch.float16 if a.dtype == "f16" else torch.float32
    p = iq.iq_make_params(a.d, a.bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    x = iqsynth.device_unit_vectors(a.n, a.d, 3, tdt, "cuda")
    ref = x.float().norm(dim=1)
    c0, n0 = iq.iq_quantize(p, x)
    y2, c2, n2 = iq.iq_roundtrip(p, x, emit_codes=True)
    torch.cuda.synchronize()
    for name, nn in (("quantize", n0), ("roundtrip+codes", n2)):
        rel = ((nn - ref).abs() / ref).cpu()
        bad = (rel > 1e-5).nonzero().flatten()
        print(name, "max rel", rel.max().item(), "bad rows", bad.numel(), bad[:16].tolist())
        if bad.numel():
            r = bad[0].item()
            print("   row", r, "tile(64)", r // 64, "in-tile", r % 64, "lib", nn[r].item(), "ref", ref[r].item())
    print("codes equal", torch.equal(c0, c2), "norms equal", torch.equal(n0, n2))


if __name__ == "__main__" and "--repeat" not in sys.argv:
    main()


def repeat_check(d=128, bits=4, n=1 << 20, reps=30, dtype="f16"):
    """Run each kernel `reps` times on the same input; any difference between
    runs reveals a race (the kernels are deterministic by construction)."""
    import torch
    import iqsynth
    import paper_2603_28430_b200 as iq
    tdt = torch.float16 if dtype == "f16" else torch.float32
    p = iq.iq_make_params(d, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    x = iqsynth.device_unit_vectors(n, d, 3, tdt, "cuda")
    ref = x.float().norm(dim=1)
    y0, c0, n0 = iq.iq_roundtrip(p, x, emit_codes=True)
    q0, qn0 = iq.iq_quantize(p, x)
    r0 = iq.iq_roundtrip(p, x)
    d0 = iq.iq_dequantize(p, q0, qn0, dtype=tdt)
    bad = {"rte": 0, "q": 0, "rt": 0, "dq": 0}
    for _ in range(reps):
        y, c, nn = iq.iq_roundtrip(p, x, emit_codes=True)
        bad["rte"] += int((~(y == y0).all(dim=1) | ~(c == c0).all(dim=1) | (nn != n0)).sum())
        q, qn = iq.iq_quantize(p, x)
        bad["q"] += int((~(q == q0).all(dim=1) | (qn != qn0)).sum())
        bad["rt"] += int((~(iq.iq_roundtrip(p, x) == r0).all(dim=1)).sum())
        bad["dq"] += int((~(iq.iq_dequantize(p, q0, qn0, dtype=tdt) == d0).all(dim=1)).sum())
    torch.cuda.synchronize()
    rel = ((n0 - ref).abs() / ref)
    print(f"d={d} b={bits} {dtype}: rows differing across {reps} reruns {bad}; first-run norm max rel {rel.max().item():.2e}")


if __name__ == "__main__" and "--repeat" in sys.argv:
    for cfg in [(128, 4, "f16"), (128, 3, "f16"), (512, 3, "f16"), (128, 3, "f32")]:
        repeat_check(d=cfg[0], bits=cfg[1], dtype=cfg[2])
