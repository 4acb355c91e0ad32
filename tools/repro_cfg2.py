import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import iqsynth, iq_parity as parity
import paper_2603_28430_b200 as iq
from oracle import iq_oracle as O
d, bits, n = 128, 4, 1 << 20
seed = iqsynth.data_seed(2, d + bits)
for variant in (0,):
    p = iq.iq_make_params(d, bits, variant, iqsynth.PARAMS_SEED, device=0)
    x = iqsynth.device_unit_vectors(n, d, seed, torch.float16, "cuda")
    rows = iqsynth.sample_rows(n, 8192, seed)
    ridx = torch.from_numpy(rows).cuda()
    X = x.index_select(0, ridx).cpu().numpy()
    y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
    torch.cuda.synchronize()
    N = norms.index_select(0, ridx).cpu().numpy()
    ref = np.linalg.norm(X.astype(np.float64), axis=1)
    rel = np.abs(N - ref) / ref
    bad = np.where(rel > 1e-5)[0]
    print("bad sample rows", len(bad), bad[:10], rows[bad[:10]])
    tn = x.float().norm(dim=1).cpu().numpy()
    allbad = np.where(np.abs(norms.cpu().numpy() - tn) / tn > 1e-5)[0]
    print("bad rows over all n (vs torch):", len(allbad), allbad[:10])
    if len(bad):
        r = rows[bad[0]]
        print("row", r, "X norm", ref[bad[0]], "torch norm of x[r]", tn[r], "gpu norm", N[bad[0]])
        print("x[r] first 8", x[r, :8].float().cpu().numpy(), "X first 8", X[bad[0], :8].astype(np.float32))
    nn = norms.cpu().numpy()
    for r in allbad[:10]:
        xr = x[r].float().cpu().numpy()
        print(f"row {r} tile {r//64} in {r%64}  gpu {nn[r]:.7f} torch {tn[r]:.7f}  rel {abs(nn[r]-tn[r])/tn[r]:.2e}  min|x| {np.abs(xr).min():.2e} max|x| {np.abs(xr).max():.3f}")
    # same rows through quantize and the value-only kernel
    q, qn = iq.iq_quantize(p, x)
    print("quantize norms at bad rows", qn.cpu().numpy()[allbad[:5]])
    # rerun roundtrip+codes on just those rows
    sub = x[torch.from_numpy(allbad).cuda()].contiguous()
    ys, cs, ns = iq.iq_roundtrip(p, sub, emit_codes=True)
    print("isolated rerun norms", ns.cpu().numpy()[:5], "torch", tn[allbad[:5]])
