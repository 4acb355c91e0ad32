"""For rows whose norm is wrong, find which input row's norm the kernel
actually produced (identifies a stage overwritten by a later tile vs stale
shared memory)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import iqsynth
import paper_2603_28430_b200 as iq
kind = sys.argv[1]
d, bits, n = 128, int(sys.argv[2]) if len(sys.argv) > 2 else 4, 1 << 20
seed = iqsynth.data_seed(2, 132)
p = iq.iq_make_params(d, bits, 0, iqsynth.PARAMS_SEED, device=0)
x = iqsynth.device_unit_vectors(n, d, seed, torch.float16, "cuda")
rows = iqsynth.sample_rows(n, 8192, seed)
X = x.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
for rep in range(3):
    if kind == "rte":
        y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
    else:
        codes, norms = iq.iq_quantize(p, x)
    torch.cuda.synchronize()
    tn = x.float().norm(dim=1)
    rel = (norms - tn).abs() / tn
    bad = (rel > 1e-5).nonzero().flatten().tolist()
    print(f"rep {rep} bad {len(bad)}", flush=True)
    tnc = tn.cpu().numpy()
    for r in bad[:12]:
        v = norms[r].item()
        cand = np.nonzero(np.abs(tnc - v) <= 3e-7 * v)[0]
        cand = cand[np.argsort(np.abs(cand - r))][:4]
        print(f"  row {r} tile {r//64} in {r%64} lib {v:.8f} ref {tnc[r]:.8f} matches {cand.tolist()} deltas {[int(c)-r for c in cand]}", flush=True)
