"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs, element by element, with the north-star tolerances
(tests/parity.py).  Needs a B200 (sm_100a)."""
import math

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

NP = {iq.F32: np.float32, iq.F16: np.float16}
TT = {iq.F32: torch.float32, iq.F16: torch.float16}
SEED = iqsynth.PARAMS_SEED


def _run_all(p, X, dt):
    x = torch.from_numpy(X).cuda()
    y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
    y_plain = iq.iq_roundtrip(p, x)
    cq, nq = iq.iq_quantize(p, x)
    ydq = iq.iq_dequantize(p, cq, nq, dtype=TT[dt])
    torch.cuda.synchronize()
    return (y.cpu().numpy(), codes.cpu().numpy(), norms.cpu().numpy(), y_plain.cpu().numpy(),
            cq.cpu().numpy(), nq.cpu().numpy(), ydq.cpu().numpy())


def _parity(variant, dt, d, bits, X, seed=SEED):
    """Every stage-1 kernel's own output against the oracle, no row exempt:
    the fused kernel as benchmarked (MODE 1, value only) through its implied
    codes, the fused kernel with codes (MODE 2) and the quantizer (K1) through
    their codes and norms, the dequantizer (K2) against the oracle's decode
    of the quantizer's codes."""
    p = iq.iq_make_params(d, bits, variant, seed, device=0)
    po = O.make_params(d, bits, variant, seed)
    y, codes, norms, y_plain, cq, nq, ydq = _run_all(p, X, dt)
    # the ABI promises that quantize and the fused kernel with codes emit
    # identical codes and norms (one decision rule, one geometry)
    assert np.array_equal(codes, cq) and np.array_equal(norms, nq)
    check_mse = X.shape[0] >= 256
    r = parity.check(X, po, y, codes, norms, NP[dt])                 # K3 + codes, K1
    parity.assert_parity(r, NP[dt], check_mse=check_mse)
    rv = parity.check_values(X, po, y_plain, NP[dt])                 # K3 (bench.py's kernel)
    parity.assert_values(rv, NP[dt], check_mse=check_mse)
    assert parity.check_decode(cq, nq, ydq, po) <= parity.RECON_RTOL[NP[dt]]   # K2
    return r


@pytest.mark.parametrize("dt", [iq.F32, iq.F16])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d", [64, 128, 256, 512])
@pytest.mark.parametrize("bits", [1, 2, 3, 4])
def test_parity_grid(variant, dt, d, bits):
    n = 4096 if d <= 256 else 2048
    X = iqsynth.unit_vectors(n, d, iqsynth.data_seed(1, d * 10 + bits), NP[dt])
    _parity(variant, dt, d, bits, X)


@pytest.mark.parametrize("n", [1, 2, 31, 33, 257, 4095])
@pytest.mark.parametrize("dt", [iq.F32, iq.F16])
def test_ragged_n(n, dt):
    X = iqsynth.unit_vectors(n, 128, 77 + n, NP[dt])
    _parity(iq.FULL, dt, 128, 3, X)
    X = iqsynth.unit_vectors(n, 512, 78 + n, NP[dt])
    _parity(iq.FAST, dt, 512, 2, X)


@pytest.mark.parametrize("dt", [iq.F32, iq.F16])
def test_edge_vectors(dt):
    """Zero rows (x^ = 0 exactly), un-normalised rows with large / small
    norms, a row with a single nonzero, and outlier-channel rows."""
    d = 128
    X = np.concatenate([
        np.zeros((3, d)),
        iqsynth.gaussian_rows(40, d, 5, np.float64, sigma=30.0),
        iqsynth.gaussian_rows(40, d, 6, np.float64, sigma=1e-3),
        np.eye(d)[:5] * 0.5,
        iqsynth.outlier_vectors(40, d, 7, np.float64),
    ]).astype(NP[dt])
    r = _parity(iq.FULL, dt, d, 3, X)
    p = iq.iq_make_params(d, 3, iq.FULL, SEED, device=0)
    y = iq.iq_roundtrip(p, torch.from_numpy(X).cuda()).cpu().numpy()
    assert np.all(y[:3] == 0)
    assert r.n_code_mismatch <= 1


def test_bits4_all_variants_fp32():
    X = iqsynth.unit_vectors(512, 128, 9, np.float32)
    for v in (iq.FULL, iq.FAST, iq.PLANAR2D):
        _parity(v, iq.F32, 128, 4, X)


def test_in_place_roundtrip():
    X = iqsynth.unit_vectors(1000, 256, 10, np.float16)
    p = iq.iq_make_params(256, 3, iq.FAST, SEED, device=0)
    x = torch.from_numpy(X).cuda()
    y_ref = iq.iq_roundtrip(p, x)
    x2 = x.clone()
    iq.iq_roundtrip(p, x2, y=x2)
    assert torch.equal(x2, y_ref)


def test_zero_n_and_errors():
    p = iq.iq_make_params(128, 3, iq.FULL, SEED, device=0)
    x = torch.empty((0, 128), dtype=torch.float16, device="cuda")
    assert iq.iq_roundtrip(p, x).shape == (0, 128)
    xb = torch.zeros((4, 129), dtype=torch.float16, device="cuda")
    with pytest.raises(ValueError):
        iq.iq_roundtrip(p, xb)
    raw = torch.zeros(4 * 128 + 8, dtype=torch.float16, device="cuda")
    mis = raw[1:1 + 4 * 128].view(4, 128)
    with pytest.raises(iq.IQError) as e:
        iq.iq_roundtrip(p, mis)
    assert e.value.status == 3   # IQ_ERR_MISALIGNED
    with pytest.raises(iq.IQError) as e:
        iq.iq_make_params(100, 3, iq.FULL, SEED, device=0)
    assert e.value.status == 2   # IQ_ERR_UNSUPPORTED


def test_error_sums_kernel():
    X = iqsynth.unit_vectors(3000, 128, 12, np.float16)
    p = iq.iq_make_params(128, 3, iq.FULL, SEED, device=0)
    x = torch.from_numpy(X).cuda()
    y = iq.iq_roundtrip(p, x)
    s = iq.iq_error_sums(p, x, y).cpu().numpy()
    x64, y64 = X.astype(np.float64), y.cpu().numpy().astype(np.float64)
    assert s[0] == pytest.approx(np.sum((x64 - y64) ** 2), rel=1e-5)
    assert s[1] == pytest.approx(np.sum(x64 ** 2), rel=1e-5)


def test_host_pipeline_matches_device_path():
    X = iqsynth.unit_vectors(50000, 128, 13, np.float16)
    p = iq.iq_make_params(128, 3, iq.FULL, SEED, device=0)
    xh = torch.from_numpy(X).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    codes = torch.empty((50000, 48), dtype=torch.uint8).pin_memory()
    norms = torch.empty(50000, dtype=torch.float32).pin_memory()
    pl = iq.HostPipeline(p, iq.F16, chunk_vectors=4096)
    pl.roundtrip(xh, yh, codes, norms)
    yd, cd, nd = iq.iq_roundtrip(p, xh.cuda(), emit_codes=True)
    assert torch.equal(yh, yd.cpu()) and torch.equal(codes, cd.cpu()) and torch.equal(norms, nd.cpu())


def test_multi_stream_concurrency():
    """One immutable handle used from two streams at once gives the same
    results as serial calls."""
    p = iq.iq_make_params(128, 3, iq.FULL, SEED, device=0)
    xs = [torch.from_numpy(iqsynth.unit_vectors(20000, 128, 20 + i, np.float16)).cuda() for i in range(2)]
    ref = [iq.iq_roundtrip(p, x) for x in xs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [None, None]
    for i in range(2):
        with torch.cuda.stream(streams[i]):
            outs[i] = iq.iq_roundtrip(p, xs[i], stream=streams[i])
    torch.cuda.synchronize()
    for i in range(2):
        assert torch.equal(outs[i], ref[i])


# ------------------------------------------------------------ full-size configs
def _large_config(variant, dt, d, bits, n, data_seed, in_place=False, sample=65536):
    """Run at BASELINE full size on device-resident inputs (the launch
    configuration bench.py times), check a seeded row sample against the
    oracle element by element, and the full-batch MSE against the closed
    form (P:277-279 with k = d) within 5 standard errors."""
    p = iq.iq_make_params(d, bits, variant, SEED, device=0)
    x = iqsynth.device_unit_vectors(n, d, data_seed, TT[dt], "cuda")
    rows = iqsynth.sample_rows(n, sample, data_seed)
    ridx = torch.from_numpy(rows).cuda()
    X = x.index_select(0, ridx).cpu().numpy()
    if in_place:
        codes = torch.empty((n, p.code_bytes), dtype=torch.uint8, device="cuda")
        norms = torch.empty(n, dtype=torch.float32, device="cuda")
        iq.iq_roundtrip(p, x, y=x, codes=codes, norms=norms)
        y = x
        yS = y.index_select(0, ridx)
        sums = None
    else:
        y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
        sums = iq.iq_error_sums(p, x, y)
        yS = y.index_select(0, ridx)
    torch.cuda.synchronize()
    r = parity.check(X, O.make_params(d, bits, variant, SEED), yS.cpu().numpy(),
                     codes.index_select(0, ridx).cpu().numpy(), norms.index_select(0, ridx).cpu().numpy(),
                     NP[dt])
    parity.assert_parity(r, NP[dt])
    mse = None
    if sums is not None:
        s = sums.cpu().numpy()
        mse = s[0] / (n * d)
        expect = O.expected_unit_vector_mse(d, bits)
        # CV of per-vector squared error <= 0.25 -> SE bound
        se = 0.25 * expect / math.sqrt(n)
        fp16_extra = 2e-3 * expect if dt == iq.F16 else 0.0
        assert abs(mse - expect) <= 5 * se + fp16_extra + 1e-4 * expect, (mse, expect)
    del x, y, codes, norms
    torch.cuda.empty_cache()
    return r, mse


def _bench_launch_parity(variant, dt, d, bits, n, config=2, steps=6, sample=65536):
    """The kernel bench.py times, in the launch configuration it times it:
    iq_roundtrip WITHOUT codes (the fused MODE-1 instance) over the bench's
    two rotating device buffers (iqsynth.dist.rank_buffers, the same seeds),
    launched back to back on one stream; then a seeded sample of each
    buffer's output rows against the oracle through check_values, no row
    exempt."""
    from iqsynth import dist as D
    p = iq.iq_make_params(d, bits, variant, SEED, device=0)
    xs, _, _ = D.rank_buffers(config, n, d, TT[dt], "cuda")
    ys = [torch.empty_like(x) for x in xs]
    stream = torch.cuda.current_stream()
    for i in range(steps):
        iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], stream=stream)
    torch.cuda.synchronize()
    po = O.make_params(d, bits, variant, SEED)
    for j in range(2):
        rows = iqsynth.sample_rows(n, sample, 7 + j)
        ridx = torch.from_numpy(rows).cuda()
        X = xs[j].index_select(0, ridx).cpu().numpy()
        Y = ys[j].index_select(0, ridx).cpu().numpy()
        parity.assert_values(parity.check_values(X, po, Y, NP[dt]), NP[dt])
    del xs, ys
    torch.cuda.empty_cache()


def test_bench_kernel_headline_full_d128_b3_fp16_1M():
    """BASELINE configs[1] headline, exactly as bench.py runs it."""
    _bench_launch_parity(iq.FULL, iq.F16, 128, 3, 1 << 20)


@pytest.mark.parametrize("variant,dt,d,bits", [(iq.FAST, iq.F16, 512, 4), (iq.FULL, iq.F32, 256, 2),
                                               (iq.FAST, iq.F16, 128, 4), (iq.PLANAR2D, iq.F16, 256, 2)])
def test_bench_kernel_other_settings_1M(variant, dt, d, bits):
    _bench_launch_parity(variant, dt, d, bits, 1 << 20, sample=16384)


def test_cfg2_headline_full_d128_b3_fp16_1M():
    _large_config(iq.FULL, iq.F16, 128, 3, 1 << 20, iqsynth.data_seed(2))


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("d", [128, 256, 512])
@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST])
def test_cfg2_grid_1M(variant, bits, d, dt):
    _large_config(variant, dt, d, bits, 1 << 20, iqsynth.data_seed(2, d + bits), sample=8192)


def test_cfg3_kv_cache_fast_d128_b4_fp16():
    _large_config(iq.FAST, iq.F16, 128, 4, 32 * 8 * 32768, iqsynth.data_seed(3))


def test_cfg4_planar_d256_b2_fp16_16M_and_variants_agree():
    """configs[3]: 2D, Full and Fast on the SAME 16M inputs; each against the
    oracle on a row sample and the closed form, and their full-batch MSEs
    equal to each other within the Monte Carlo error of the difference of two
    independent estimates (the paper's 'indistinguishable' MSEs)."""
    n = 1 << 24
    mses = {}
    for v in (iq.PLANAR2D, iq.FULL, iq.FAST):
        _, mses[v] = _large_config(v, iq.F16, 256, 2, n, iqsynth.data_seed(4))
    expect = O.expected_unit_vector_mse(256, 2)
    se_diff = math.sqrt(2.0) * 0.25 * expect / math.sqrt(n)
    for v in (iq.FULL, iq.FAST):
        assert abs(mses[v] - mses[iq.PLANAR2D]) <= 5 * se_diff + 2e-3 * expect, mses


def test_cfg5_full_d512_b2_fp16_64M_in_place():
    free, _ = torch.cuda.mem_get_info()
    n = 1 << 26
    if free < n * 512 * 2 * 1.2:
        pytest.skip("not enough device memory for 64 GiB")
    _large_config(iq.FULL, iq.F16, 512, 2, n, iqsynth.data_seed(5), in_place=True)


@pytest.mark.parametrize("d,bits,dt", [(128, 4, iq.F16), (512, 4, iq.F16), (512, 3, iq.F32), (128, 3, iq.F16)])
def test_norms_over_many_fresh_launches(d, bits, dt):
    """Regression for a warp-divergence bug: every row's norm from every
    encoder kernel equals torch's row norm to fp32 rounding, over many fresh
    launches (each CTA's first TMA stage is where lanes leave the mbarrier
    wait at different times)."""
    p = iq.iq_make_params(d, bits, iq.FULL, SEED, device=0)
    bad = 0
    for s in range(25):
        x = iqsynth.device_unit_vectors(16384, d, 500 + s, TT[dt], "cuda")
        tn = x.float().norm(dim=1)
        _, nq = iq.iq_quantize(p, x)
        _, _, ne = iq.iq_roundtrip(p, x, emit_codes=True)
        bad += int(((nq - tn).abs() / tn > 1e-5).sum()) + int(((ne - tn).abs() / tn > 1e-5).sum())
    assert bad == 0


@pytest.mark.gpu
def test_quantize_outputs_at_4_byte_alignment():
    """The ABI promises codes and norms need only 4-byte alignment for
    iq_quantize / iq_roundtrip (include/isoquant.h): outputs at a 4-byte
    offset equal the 16-byte-aligned ones, bit for bit."""
    for d, bits, dt in ((128, 3, np.float16), (64, 4, np.float32), (256, 2, np.float16)):
        n = 1000
        X = iqsynth.unit_vectors(n, d, 21, dt)
        x = torch.from_numpy(X).cuda()
        p = iq.iq_make_params(d, bits, iq.FULL, SEED, device=0)
        cb = p.code_bytes
        c0 = torch.empty((n, cb), dtype=torch.uint8, device="cuda")
        r0 = torch.empty(n, dtype=torch.float32, device="cuda")
        iq.iq_quantize(p, x, c0, r0)
        craw = torch.zeros(n * cb + 16, dtype=torch.uint8, device="cuda")
        rraw = torch.zeros(n + 4, dtype=torch.float32, device="cuda")
        c1 = craw[4:4 + n * cb].view(n, cb)
        r1 = rraw[1:1 + n]
        iq.iq_quantize(p, x, c1, r1)
        assert torch.equal(c0, c1) and torch.equal(r0, r1)
        y1 = torch.empty_like(x)
        c2, r2 = craw[8:8 + n * cb].view(n, cb), rraw[3:3 + n]
        iq.iq_roundtrip(p, x, y=y1, codes=c2, norms=r2)
        assert torch.equal(c0, c2) and torch.equal(r0, r2)
