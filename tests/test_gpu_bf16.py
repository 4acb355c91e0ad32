"""bfloat16 storage (R28): the same kernels with
bf16 rows in and out, against the fp64 oracle on the stored (bf16) values.
Codes and norms follow the north-star bounds unchanged (the kernels compute in
fp32); reconstructions within 8e-3 relative per row (output rounding 2^-9)."""
import numpy as np
import pytest

import iqsynth
from oracle import iq_oracle as O
import iq_parity as parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_28430_b200 as iq  # noqa: E402

SEED = iqsynth.PARAMS_SEED


def _bf16_rows(n, d, seed):
    x = torch.from_numpy(iqsynth.unit_vectors(n, d, seed, np.float32)).to(torch.bfloat16).cuda()
    return x, x.float().cpu().numpy()


@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d", [64, 128, 256, 512])
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_bf16_parity(variant, d, bits):
    n = 2048 + 33
    x, X = _bf16_rows(n, d, 900 + d + bits)
    p = iq.iq_make_params(d, bits, variant, SEED, device=0)
    po = O.make_params(d, bits, variant, SEED)
    y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
    y2 = iq.iq_roundtrip(p, x)
    cq, nq = iq.iq_quantize(p, x)
    ydq = iq.iq_dequantize(p, cq, nq, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(codes, cq) and torch.equal(norms, nq)
    r = parity.check(X, po, y.float().cpu().numpy(), codes.cpu().numpy(), norms.cpu().numpy(), "bf16")
    parity.assert_parity(r, "bf16")
    # the fused kernel without codes (through its implied codes) and the
    # decoder (against the oracle's decode of the quantizer's codes), no row exempt
    parity.assert_values(parity.check_values(X, po, y2.float().cpu().numpy(), "bf16"), "bf16")
    assert parity.check_decode(cq.cpu().numpy(), nq.cpu().numpy(), ydq.float().cpu().numpy(), po) \
        <= parity.RECON_RTOL["bf16"]


def test_bf16_sketch_and_attention():
    d = 128
    x, X = _bf16_rows(1024, d, 7)
    p = iq.iq_make_params_qjl(d, 3, iq.FULL, SEED, device=0)
    codes, norms, qjl, rn = iq.iq_quantize_qjl(p, x)
    cq, nq = iq.iq_quantize(p, x)
    assert torch.equal(codes, cq) and torch.equal(norms, nq)
    q = torch.randn((1, 4, d), dtype=torch.bfloat16, device="cuda")
    sc = iq.iq_attention_scores(p, codes.view(1, 1024, -1), norms.view(1, 1024), q, qjl.view(1, 1024, -1),
                                rn.view(1, 1024))
    torch.cuda.synchronize()
    assert torch.isfinite(sc).all()
    po = O.make_params(d, 3, iq.FULL, SEED)
    xh = O.decode(O.unpack_codes(codes.cpu().numpy(), 3, d), norms.cpu().numpy().astype(np.float64), po)
    want = q[0].float().cpu().numpy().astype(np.float64) @ xh.T
    s1 = iq.iq_attention_scores(p, codes.view(1, 1024, -1), norms.view(1, 1024), q)[0].cpu().numpy()
    qn = np.linalg.norm(q[0].float().cpu().numpy(), axis=1)[:, None]
    assert np.all(np.abs(s1 - want) <= 2e-3 * qn * norms.cpu().numpy()[None, :] + 1e-30)


def test_bf16_error_sums_and_host_pipeline():
    d = 128
    x, X = _bf16_rows(4096, d, 8)
    p = iq.iq_make_params(d, 3, iq.FULL, SEED, device=0)
    y = iq.iq_roundtrip(p, x)
    sums = iq.iq_error_sums(p, x, y)
    want = float(((x.double() - y.double()) ** 2).sum())
    assert abs(float(sums[0]) - want) <= 1e-6 * want
    pl = iq.HostPipeline(p, iq.BF16, chunk_vectors=1000)
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    pl.roundtrip(xh, yh)
    assert torch.equal(yh, y.cpu())
