"""GPU parity of the fused KV-cache decode consumer (iq_attention_scores,
tcgen05) against the CPU oracle (oracle/attn_oracle.py) on the GPU's own
codes.  Tolerance (R27, from the arithmetic): fp16 centroids and
fp16 rotated queries (power-of-two scaled) give |error| <= 2e-3 rho_k ||q_j||
for the stage-1 logit; the stage-2 term adds fp16 S q (each element within
2^-11 ||S_i|| ||q||) summed over m signs: <= 2e-3 sqrt(d) gamma_k ||q_j||."""
import numpy as np
import pytest

import iqsynth
from oracle import attn_oracle as A
from oracle import iq_oracle as O
from oracle import qjl_oracle as Q

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_28430_b200 as iq  # noqa: E402

SEED = iqsynth.PARAMS_SEED
TT = {iq.F32: torch.float32, iq.F16: torch.float16}
NP = {iq.F32: np.float32, iq.F16: np.float16}
_S = {}


def _run(d, bits, variant, dt, heads, n_keys, n_q, stage2, seed=0):
    mk = iq.iq_make_params_qjl if stage2 else iq.iq_make_params
    p = mk(d, bits, variant, SEED, device=0)
    X = iqsynth.unit_vectors(heads * n_keys, d, 700 + seed, NP[dt])
    X = (X.astype(np.float32) * np.float32(1.5)).astype(NP[dt])
    x = torch.from_numpy(X).cuda()
    if stage2:
        codes, norms, qjl, rn = iq.iq_quantize_qjl(p, x)
        qjl, rn = qjl.view(heads, n_keys, -1), rn.view(heads, n_keys)
    else:
        codes, norms = iq.iq_quantize(p, x)
        qjl = rn = None
    codes, norms = codes.view(heads, n_keys, -1), norms.view(heads, n_keys)
    Qh = (np.random.default_rng(seed).standard_normal((heads, n_q, d)) * 3).astype(NP[dt])
    q = torch.from_numpy(Qh).cuda()
    sc = iq.iq_attention_scores(p, codes, norms, q, qjl, rn)
    torch.cuda.synchronize()
    sc = sc.cpu().numpy().astype(np.float64)
    po = O.make_params(d, bits, variant, SEED)
    w = O.block_width(variant)
    mpad = -(-d // w) * w
    S = None
    if stage2:
        if d not in _S:
            _S[d] = Q.sketch_matrix(d, SEED)
        S = _S[d]
    cn, nn = codes.cpu().numpy(), norms.cpu().numpy().astype(np.float64)
    for h in range(heads):
        cu = O.unpack_codes(cn[h], bits, mpad)
        Qf = Qh[h].astype(np.float64)
        if stage2:
            q01 = Q.unpack_bits(qjl[h].cpu().numpy(), d)
            g = rn[h].cpu().numpy().astype(np.float64)
            want = A.attention_scores(Qf, cu, nn[h], po, q01, g, S)
        else:
            g = np.zeros(n_keys)
            want = A.attention_scores(Qf, cu, nn[h], po)
        qn = np.linalg.norm(Qf, axis=1)[:, None]
        tol = 2e-3 * nn[h][None, :] * qn + 2e-3 * np.sqrt(d) * g[None, :] * qn + 1e-30
        err = np.abs(sc[h] - want)
        assert np.all(err <= tol), (h, float(np.max(err / tol)))
    return sc


@pytest.mark.parametrize("stage2", [False, True])
@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_attn_grid(bits, d, dt, stage2):
    _run(d, bits, iq.FULL, dt, heads=2, n_keys=1024 + 4 * bits, n_q=4, stage2=stage2, seed=bits)


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d", [256, 512])
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_attn_wide_heads(bits, d, variant, dt):
    """d in {256, 512} (the paper's widths): the key tile's A operand
    is built and accumulated in 128-coordinate chunks (stage 1)."""
    _run(d, bits, variant, dt, heads=3, n_keys=700 + 4 * bits, n_q=5, stage2=False, seed=d + bits)


@pytest.mark.parametrize("n_keys", [1, 129, 4100])
def test_attn_wide_shapes_and_head_switches(n_keys):
    _run(512, 4, iq.FULL, iq.F16, heads=1, n_keys=n_keys, n_q=16, stage2=False, seed=n_keys)
    _run(256, 3, iq.FAST, iq.F16, heads=300, n_keys=128, n_q=4, stage2=False, seed=3)


@pytest.mark.parametrize("bits", [2, 3])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
def test_attn_stage2_d256(variant, bits):
    """The stage-2 term at d = 256 (b <= 3): S q over two 128-row tiles of S,
    the sketch-bit operand in two K-chunks; ragged keys, several heads."""
    _run(256, bits, variant, iq.F16, heads=3, n_keys=300, n_q=5, stage2=True, seed=17 + bits)


@pytest.mark.parametrize("d,bits", [(256, 4), (512, 2)])
def test_attn_wide_stage2_unsupported(d, bits):
    p = iq.iq_make_params(d, bits, iq.FULL, SEED, device=0)
    cb = d * bits // 8
    codes = torch.zeros((1, 8, cb), dtype=torch.uint8, device="cuda")
    norms = torch.zeros((1, 8), dtype=torch.float32, device="cuda")
    qjl = torch.zeros((1, 8, d // 8), dtype=torch.uint8, device="cuda")
    q = torch.zeros((1, 2, d), dtype=torch.float16, device="cuda")
    with pytest.raises(iq.IQError):
        iq.iq_attention_scores(p, codes, norms, q, qjl, norms.clone())


@pytest.mark.parametrize("variant", [iq.FAST, iq.PLANAR2D])
def test_attn_variants(variant):
    _run(128, 3, variant, iq.F16, heads=3, n_keys=600, n_q=8, stage2=True, seed=11)


@pytest.mark.parametrize("n_q", [1, 16])
@pytest.mark.parametrize("n_keys", [1, 127, 129, 4100])
def test_attn_shapes(n_keys, n_q):
    _run(128, 3, iq.FULL, iq.F16, heads=1, n_keys=n_keys, n_q=n_q, stage2=True, seed=n_keys)


def test_attn_many_heads_head_switches():
    """More heads than SMs: every CTA switches heads (query re-preparation)."""
    _run(64, 2, iq.FULL, iq.F16, heads=300, n_keys=256, n_q=4, stage2=True, seed=5)


def test_attn_errors():
    p = iq.iq_make_params(128, 3, iq.FULL, SEED, device=0)
    codes = torch.zeros((2, 8, 48), dtype=torch.uint8, device="cuda")
    norms = torch.zeros((2, 8), dtype=torch.float32, device="cuda")
    q = torch.zeros((2, 17, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(iq.IQError):
        iq.iq_attention_scores(p, codes, norms, q)                         # n_q > 16
    qj = torch.zeros((2, 8, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(iq.IQError):
        iq.iq_attention_scores(p, codes, norms, q[:, :4].contiguous(), qj, norms)   # no sketch in handle
    codes6 = torch.zeros((2, 6, 48), dtype=torch.uint8, device="cuda")
    with pytest.raises(iq.IQError):
        iq.iq_attention_scores(p, codes6, norms[:, :6].contiguous(), q[:, :4].contiguous())   # 6 % 4 != 0


def test_attn_kv_cache_shaped_sample():
    """configs[2] shape (32 layers x 8 KV heads x 32768 tokens, Fast d=128
    b=4 fp16, 4 queries per KV head) in one launch with the stage-2 sketch;
    sampled heads and keys against the oracle."""
    d, bits, heads, n_keys = 128, 4, 32 * 8, 32768
    p = iq.iq_make_params_qjl(d, bits, iq.FAST, SEED, device=0)
    n = heads * n_keys
    codes = torch.empty((n, p.code_bytes), dtype=torch.uint8, device="cuda")
    norms = torch.empty(n, dtype=torch.float32, device="cuda")
    qj = torch.empty((n, d // 8), dtype=torch.uint8, device="cuda")
    rn = torch.empty(n, dtype=torch.float32, device="cuda")
    chunk = 1 << 22
    for r0 in range(0, n, chunk):
        x = iqsynth.device_unit_vectors(chunk, d, 600 + r0 // chunk, torch.float16, "cuda")
        iq.iq_quantize_qjl(p, x, codes[r0:r0 + chunk], norms[r0:r0 + chunk], qj[r0:r0 + chunk], rn[r0:r0 + chunk])
    del x
    q = torch.randn((heads, 4, d), dtype=torch.float16, device="cuda")
    sc = iq.iq_attention_scores(p, codes.view(heads, n_keys, -1), norms.view(heads, n_keys), q,
                                qj.view(heads, n_keys, -1), rn.view(heads, n_keys))
    torch.cuda.synchronize()
    po = O.make_params(d, bits, iq.FAST, SEED)
    S = Q.sketch_matrix(d, SEED)
    rng = np.random.default_rng(2)
    for h in (0, 137, heads - 1):
        ks = np.sort(rng.choice(n_keys, 512, replace=False))
        rows = torch.from_numpy(h * n_keys + ks).cuda()
        cu = O.unpack_codes(codes[rows].cpu().numpy(), bits, d)
        g = rn[rows].cpu().numpy().astype(np.float64)
        nn = norms[rows].cpu().numpy().astype(np.float64)
        Qf = q[h].float().cpu().numpy().astype(np.float64)
        want = A.attention_scores(Qf, cu, nn, po, Q.unpack_bits(qj[rows].cpu().numpy(), d), g, S)
        got = sc[h][:, torch.from_numpy(ks).cuda()].cpu().numpy()
        qn = np.linalg.norm(Qf, axis=1)[:, None]
        tol = 2e-3 * nn[None, :] * qn + 2e-3 * np.sqrt(d) * g[None, :] * qn
        assert np.all(np.abs(got - want) <= tol)
