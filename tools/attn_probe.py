"""Run the decode consumer once per (d, bits) on small synthetic caches
(debug helper: python tools/attn_probe.py [d bits heads keys])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import iqsynth  # noqa: E402
import paper_2603_28430_b200 as iq  # noqa: E402

cases = [(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))] if len(sys.argv) > 4 else \
    [(d, b, 3, 708) for d in (256, 512) for b in (2, 3, 4)]
for d, b, heads, keys in cases:
    p = iq.iq_make_params(d, b, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    x = iqsynth.device_unit_vectors(heads * keys, d, 5, torch.float16, "cuda")
    codes, norms = iq.iq_quantize(p, x)
    q = torch.randn((heads, 4, d), dtype=torch.float16, device="cuda")
    sc = iq.iq_attention_scores(p, codes.view(heads, keys, -1), norms.view(heads, keys), q)
    torch.cuda.synchronize()
    print(d, b, "ok", float(sc.abs().max()), flush=True)
