"""Parameter sets (R31): one handle with n_sets rotation
sets, row r using set (r // set_rows) % n_sets and head h of the consumer
set h % n_sets; every kernel against the oracle built with the matching
per-set parameters (seed + s)."""
import numpy as np
import pytest

import iqsynth
from oracle import attn_oracle as A
from oracle import iq_oracle as O
import iq_parity as parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_28430_b200 as iq  # noqa: E402

SEED = iqsynth.PARAMS_SEED
NP = {iq.F32: np.float32, iq.F16: np.float16}
TT = {iq.F32: torch.float32, iq.F16: torch.float16}


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d,bits", [(64, 2), (128, 3), (128, 4), (256, 3), (512, 2)])
def test_sets_stage1(d, bits, variant, dt):
    n_sets, set_rows = 3, 256
    n = 2 * n_sets * set_rows + 37                       # wraps around the sets, ragged tail
    X = iqsynth.unit_vectors(n, d, 31 + d + bits, NP[dt])
    p = iq.iq_make_params_sets(d, bits, variant, SEED, n_sets, set_rows, device=0)
    x = torch.from_numpy(X).cuda()
    y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
    cq, nq = iq.iq_quantize(p, x)
    ydq = iq.iq_dequantize(p, cq, nq, dtype=TT[dt])
    torch.cuda.synchronize()
    assert torch.equal(codes, cq) and torch.equal(norms, nq)
    y, codes, norms, ydq = y.cpu().numpy(), codes.cpu().numpy(), norms.cpu().numpy(), ydq.cpu().numpy()
    set_of_row = (np.arange(n) // set_rows) % n_sets
    for s in range(n_sets):
        rows = set_of_row == s
        po = O.make_params(d, bits, variant, SEED + s)
        r = parity.check(X[rows], po, y[rows], codes[rows], norms[rows], NP[dt])
        parity.assert_parity(r, NP[dt])
        r = parity.check(X[rows], po, ydq[rows], codes[rows], norms[rows], NP[dt])
        assert r.max_recon_rel_all <= parity.RECON_RTOL[NP[dt]], r


def test_sets_attention_per_head():
    d, bits, heads, n_keys = 128, 3, 4, 512
    n_sets = 2
    p = iq.iq_make_params_sets(d, bits, iq.FULL, SEED, n_sets, n_keys, device=0)
    X = iqsynth.unit_vectors(heads * n_keys, d, 5, np.float16)
    codes, norms = iq.iq_quantize(p, torch.from_numpy(X).cuda())
    q = torch.randn((heads, 4, d), dtype=torch.float16, device="cuda")
    sc = iq.iq_attention_scores(p, codes.view(heads, n_keys, -1), norms.view(heads, n_keys), q)
    torch.cuda.synchronize()
    cn, nn = codes.cpu().numpy().reshape(heads, n_keys, -1), norms.cpu().numpy().reshape(heads, n_keys)
    for h in range(heads):
        po = O.make_params(d, bits, iq.FULL, SEED + h % n_sets)
        Qf = q[h].float().cpu().numpy().astype(np.float64)
        want = A.attention_scores(Qf, O.unpack_codes(cn[h], bits, d), nn[h].astype(np.float64), po)
        tol = 2e-3 * np.linalg.norm(Qf, axis=1)[:, None] * nn[h][None, :]
        assert np.all(np.abs(sc[h].cpu().numpy() - want) <= tol + 1e-30)


def test_sets_host_pipeline_and_errors():
    d, n_sets, set_rows = 128, 2, 256
    p = iq.iq_make_params_sets(d, 3, iq.FAST, SEED, n_sets, set_rows, device=0)
    X = torch.from_numpy(iqsynth.unit_vectors(4 * n_sets * set_rows, d, 9, np.float16))
    pl = iq.HostPipeline(p, iq.F16, chunk_vectors=2 * n_sets * set_rows)
    xh = X.pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    pl.roundtrip(xh, yh)
    assert torch.equal(yh, iq.iq_roundtrip(p, X.cuda()).cpu())
    with pytest.raises(iq.IQError):
        iq.HostPipeline(p, iq.F16, chunk_vectors=300)
    with pytest.raises(iq.IQError):
        iq.iq_distortion_grad(p, X.cuda())
