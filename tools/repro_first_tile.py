"""Count rows whose norm from each encoder kernel disagrees with torch, over
many fresh launches on small inputs (first-tile behaviour)."""
import sys
import torch
sys.path.insert(0, '.')
import iqsynth
import paper_2603_28430_b200 as iq

def run(d, bits, dt, launches=40, n=16384):
    tdt = torch.float16 if dt == "f16" else torch.float32
    p = iq.iq_make_params(d, bits, 0, iqsynth.PARAMS_SEED, device=0)
    bad = {"q": 0, "rte": 0}
    for s in range(launches):
        x = iqsynth.device_unit_vectors(n, d, 100 + s, tdt, "cuda")
        tn = x.float().norm(dim=1)
        _, nq = iq.iq_quantize(p, x)
        _, _, ne = iq.iq_roundtrip(p, x, emit_codes=True)
        bad["q"] += int(((nq - tn).abs() / tn > 1e-5).sum())
        bad["rte"] += int(((ne - tn).abs() / tn > 1e-5).sum())
    print(d, bits, dt, bad, flush=True)

for cfg in [(128, 4, "f16"), (128, 3, "f16"), (128, 2, "f16"), (256, 4, "f16"), (128, 4, "f32"), (512, 4, "f16")]:
    run(*cfg)
