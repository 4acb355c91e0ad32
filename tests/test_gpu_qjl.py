"""GPU parity of the stage-2 residual sketch (iq_quantize_qjl, the tcgen05
path: one fused kernel at d in {64, 128}, quantizer + K-chunked sketch
kernel at d in {256, 512}) against the CPU oracle (oracle/qjl_oracle.py) on
the same seeded inputs.  Tolerances (R20-R24, derived from the arithmetic):
  * codes and norms bit-identical to iq_quantize (same kernel rule);
  * gamma = ||r|| within 2e-5 relative of the oracle's residual norm built
    from the GPU's own codes (x^ in fp32 vs fp64: ~1e-6 of ||r||);
  * sketch bits: >= 99.99 % agreement with the oracle's [S r >= 0] and every
    mismatch at |z| <= 1e-5 ||S_i|| ||r|| (fp32 x^, fp16 hi+lo split and fp32
    tensor-core accumulation perturb z by ~1e-6 ||S_i|| ||r||)."""
import numpy as np
import pytest

import iqsynth
from oracle import iq_oracle as O
from oracle import qjl_oracle as Q

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_28430_b200 as iq  # noqa: E402

SEED = iqsynth.PARAMS_SEED
NP = {iq.F32: np.float32, iq.F16: np.float16}
_S = {}


def _sketch(d):
    if d not in _S:
        _S[d] = Q.sketch_matrix(d, SEED)
    return _S[d]


def _check(X, d, bits, variant, dt):
    p = iq.iq_make_params_qjl(d, bits, variant, SEED, device=0)
    po = O.make_params(d, bits, variant, SEED)
    S = _sketch(d)
    assert np.array_equal(iq.iq_export_qjl_matrix(p).astype(np.float64), S)   # C++ generator == oracle's
    x = torch.from_numpy(X).cuda()
    codes, norms, qjl, rn = iq.iq_quantize_qjl(p, x)
    cq, nq = iq.iq_quantize(p, x)
    torch.cuda.synchronize()
    codes, norms, qjl, rn = (t.cpu().numpy() for t in (codes, norms, qjl, rn))
    assert np.array_equal(codes, cq.cpu().numpy()) and np.array_equal(norms, nq.cpu().numpy())
    return _verify(X, d, bits, variant, codes, qjl, rn)


def _verify(X, d, bits, variant, codes, qjl, rn):
    po = O.make_params(d, bits, variant, SEED)
    S = _sketch(d)
    # the oracle's residual for the GPU's own stage-1 codes (a rare stage-1
    # decision at a threshold then does not cascade into the sketch check)
    X64 = X.astype(np.float64)
    w = O.block_width(variant)
    mpad = -(-d // w) * w
    rho_o = np.sqrt(np.sum(X64 * X64, axis=1))
    xh = O.decode(O.unpack_codes(codes, bits, mpad), rho_o, po)
    R = X64 - xh
    g_o = np.linalg.norm(R, axis=1)
    nz = g_o > 0
    assert np.all(np.abs(rn[nz] - g_o[nz]) <= 2e-5 * g_o[nz]), np.max(np.abs(rn[nz] - g_o[nz]) / g_o[nz])
    assert np.all(rn[~nz] == 0)
    Z = R @ S.T
    bits_o = (Z >= 0).astype(np.uint8)
    bits_g = Q.unpack_bits(qjl, d)
    mism = bits_g != bits_o
    agree = 1.0 - mism.mean()
    assert agree >= 0.9999, agree
    if mism.any():
        scale = np.linalg.norm(S, axis=1)[None, :] * g_o[:, None]
        assert np.all(np.abs(Z[mism]) <= 1e-5 * scale[mism]), np.max(np.abs(Z[mism]) / scale[mism])
    return agree


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
def test_qjl_grid(variant, bits, d, dt):
    X = iqsynth.unit_vectors(4096 + 37, d, 100 + bits + d, NP[dt])    # 33 tiles, ragged tail
    _check(X, d, bits, variant, dt)


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("d", [256, 512])
@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
def test_qjl_wide_grid(variant, bits, d, dt):
    """The paper's wider heads: the quantizer + K-chunked sketch
    kernel (S streamed from L2), 17 tiles with a ragged tail."""
    X = iqsynth.unit_vectors(2048 + 37, d, 200 + bits + d, NP[dt])
    _check(X, d, bits, variant, dt)


@pytest.mark.parametrize("d", [128, 256, 512])
@pytest.mark.parametrize("n", [1, 2, 127, 128, 129, 1000])
def test_qjl_ragged(n, d):
    X = iqsynth.unit_vectors(n, d, 300 + n, np.float16)
    _check(X, d, 3, iq.FULL, iq.F16)


@pytest.mark.parametrize("d", [128, 512])
def test_qjl_special_rows(d):
    rng = np.random.default_rng(4)
    X = iqsynth.unit_vectors(512, d, 55, np.float32)
    X[0] = 0.0                              # zero row: gamma = 0, all bits +1
    X[1] *= 1e4                             # large norm
    X[2] *= 1e-3                            # small norm
    X[3] = 0.0
    X[3, 5] = 1.0                           # one-hot
    X[4:64] *= (1 + 3 * (np.arange(d) % 4 == 0))[None, :].astype(np.float32)   # outlier channels
    X[64:128] = rng.standard_normal((64, d)).astype(np.float32) * 30
    _check(X, d, 3, iq.FULL, iq.F32)
    p = iq.iq_make_params_qjl(d, 3, iq.FULL, SEED, device=0)
    _, _, qjl, rn = iq.iq_quantize_qjl(p, torch.from_numpy(X).cuda())
    assert float(rn[0]) == 0.0 and bool((qjl[0] == 0xFF).all())


@pytest.mark.parametrize("d", [128, 256, 512])
def test_qjl_large_batch_sample(d):
    """2^20 rows (the cfg2 batch) in one call; a 16384-row sample is
    checked against the oracle, and the mean of gamma^2 against the closed
    form d * E(z - Q(z))^2 of Appendix A.2."""
    bits, n = 3, 1 << 20
    p = iq.iq_make_params_qjl(d, bits, iq.FULL, SEED, device=0)
    x = iqsynth.device_unit_vectors(n, d, 4321, torch.float16, "cuda")
    codes, norms, qjl, rn = iq.iq_quantize_qjl(p, x)
    torch.cuda.synchronize()
    want = O.expected_unit_vector_mse(d, bits) * d
    got = float((rn.double() ** 2).mean())
    assert abs(got - want) <= 0.01 * want, (got, want)
    idx = torch.from_numpy(np.sort(np.random.default_rng(1).choice(n, 16384, replace=False))).cuda()
    _verify(x[idx].cpu().numpy(), d, bits, iq.FULL, codes[idx].cpu().numpy(), qjl[idx].cpu().numpy(),
            rn[idx].cpu().numpy())


def test_qjl_errors():
    p = iq.iq_make_params(128, 3, iq.FULL, SEED, device=0)
    x = torch.zeros((4, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(iq.IQError):
        iq.iq_quantize_qjl(p, x)                       # no sketch in this handle
    with pytest.raises(iq.IQError):
        iq.iq_make_params_qjl(32, 3, iq.FULL, SEED, device=0)    # GPU sketch: d in {64, 128, 256, 512}


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d,bits", [(64, 2), (128, 3), (128, 4), (256, 3), (512, 2)])
def test_qjl_sets(d, bits, variant, dt):
    """Per-(layer, head) parameter sets with the stage-2 sketch [R31]: row r
    uses set (r // set_rows) % n_sets, S is shared; codes and norms equal
    iq_quantize with the same handle, and each set's rows pass the oracle
    check built with that set's parameters (seed + s)."""
    n_sets, set_rows = 3, 256
    n = 2 * n_sets * set_rows + 37
    X = iqsynth.unit_vectors(n, d, 61 + d + bits, NP[dt])
    p = iq.iq_make_params_qjl_sets(d, bits, variant, SEED, n_sets, set_rows, device=0)
    x = torch.from_numpy(X).cuda()
    codes, norms, qjl, rn = iq.iq_quantize_qjl(p, x)
    cq, nq = iq.iq_quantize(p, x)
    torch.cuda.synchronize()
    codes, norms, qjl, rn = (t.cpu().numpy() for t in (codes, norms, qjl, rn))
    assert np.array_equal(codes, cq.cpu().numpy()) and np.array_equal(norms, nq.cpu().numpy())
    set_of_row = (np.arange(n) // set_rows) % n_sets
    S = _sketch(d)
    for s in range(n_sets):
        rows = set_of_row == s
        po = O.make_params(d, bits, variant, SEED + s)
        w = O.block_width(variant)
        mpad = -(-d // w) * w
        X64 = X[rows].astype(np.float64)
        rho_o = np.sqrt(np.sum(X64 * X64, axis=1))
        R = X64 - O.decode(O.unpack_codes(codes[rows], bits, mpad), rho_o, po)
        g_o = np.linalg.norm(R, axis=1)
        assert np.all(np.abs(rn[rows] - g_o) <= 2e-5 * g_o)
        Z = R @ S.T
        mism = Q.unpack_bits(qjl[rows], d) != (Z >= 0)
        assert mism.mean() <= 1e-4
        if mism.any():
            scale = np.linalg.norm(S, axis=1)[None, :] * g_o[:, None]
            assert np.all(np.abs(Z[mism]) <= 1e-5 * scale[mism])


def test_qjl_sets_need_256_row_sets():
    p = iq.iq_make_params_qjl_sets(128, 3, iq.FULL, SEED, 2, 128, device=0)
    x = torch.zeros((512, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(iq.IQError):
        iq.iq_quantize_qjl(p, x)
