"""Quantize-on-append into a KV cache (iq_append_kv; SURVEY 8(f) NEXT 2,
PAPER.md:460 / P:477 "fused KV-cache compression during autoregressive
decoding").  Slot r (a (layer, head) pair) appends one row per decode step
at its token position into a strided [slots, cap, code bytes] cache with
parameter set r % n_sets.  Checked against: the oracle with the slot's
per-set parameters (seed + s, R31); iq_quantize of the whole cache with
set_rows = cap (bit for bit: same lane geometry and decision code); the
decode consumer reading the appended cache; and the cache bytes it must not
touch."""
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


def _decode_steps(p, X, cap, steps, dt, positions=None):
    """Append X[:, t] (t < steps) one decode step at a time; returns the cache."""
    slots, d = X.shape[0], X.shape[2]
    codes = torch.full((slots, cap, p.code_bytes), 0xAB, dtype=torch.uint8, device="cuda")
    norms = torch.full((slots, cap), -7.0, dtype=torch.float32, device="cuda")
    x = torch.from_numpy(X).cuda()
    for t in range(steps):
        if positions is None:
            iq.iq_append_kv(p, x[:, t].contiguous(), codes, norms, position=t)
        else:
            iq.iq_append_kv(p, x[:, t].contiguous(), codes, norms, positions=positions[t])
    torch.cuda.synchronize()
    return codes, norms


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d,bits", [(64, 2), (128, 3), (128, 4), (256, 2), (512, 3), (512, 4)])
def test_append_per_head_sets_equals_batch_and_oracle(d, bits, variant, dt):
    layers, heads, cap, steps = 4, 8, 256, 5
    slots = layers * heads
    p = iq.iq_make_params_sets(d, bits, variant, SEED, slots, cap, device=0)   # one set per (layer, head)
    X = iqsynth.unit_vectors(slots * cap, d, 71 + d + bits, NP[dt]).reshape(slots, cap, d)
    codes, norms = _decode_steps(p, X, cap, steps, dt)
    # bit for bit: iq_quantize of the whole cache (row r * cap + t uses set r)
    cq, nq = iq.iq_quantize(p, torch.from_numpy(X.reshape(slots * cap, d)).cuda())
    torch.cuda.synchronize()
    cq, nq = cq.view(slots, cap, -1), nq.view(slots, cap)
    assert torch.equal(codes[:, :steps], cq[:, :steps]) and torch.equal(norms[:, :steps], nq[:, :steps])
    # nothing beyond the appended positions is touched
    assert bool((codes[:, steps:] == 0xAB).all()) and bool((norms[:, steps:] == -7.0).all())
    # against the oracle with each slot's own parameters
    cn, nn = codes.cpu().numpy(), norms.cpu().numpy()
    agree = []
    for r in range(slots):
        po = O.make_params(d, bits, variant, SEED + r)
        xh, c_o, _, rho_o = O.roundtrip(X[r, :steps], po)
        cg = O.unpack_codes(cn[r, :steps], bits, c_o.shape[1])
        mism = cg != c_o
        agree.append(mism.sum())
        if mism.any():
            y = O.rotated_coordinates(X[r, :steps], po)[mism]
            assert np.max(np.min(np.abs(y[:, None] - po.cb.thresholds[None, :]), axis=1)) <= parity.BOUNDARY
        assert np.max(np.abs(nn[r, :steps] - rho_o) / rho_o) <= parity.NORM_RTOL
    assert sum(agree) <= max(1, int(1e-4 * slots * steps * d))


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
def test_append_single_set_and_ragged_positions(dt):
    d, bits, slots, cap = 128, 3, 37, 50          # any cap (not a multiple of 256), odd slot count
    p = iq.iq_make_params(d, bits, iq.FULL, SEED, device=0)
    steps = 6
    X = iqsynth.unit_vectors(slots * steps, d, 5, NP[dt]).reshape(slots, steps, d)
    rng = np.random.default_rng(3)
    # per-slot positions: distinct lengths per sequence; some slots idle (-1) or past the cap
    pos = np.stack([rng.permutation(cap)[:steps] for _ in range(slots)], axis=1)
    pos[2, 3] = -1
    pos[4, 1] = cap + 5
    positions = [torch.from_numpy(pos[t].astype(np.int64)).cuda() for t in range(steps)]
    codes, norms = _decode_steps(p, X, cap, steps, dt, positions=positions)
    cq, nq = iq.iq_quantize(p, torch.from_numpy(X.reshape(-1, d)).cuda())
    cq, nq = cq.view(slots, steps, -1).cpu().numpy(), nq.view(slots, steps).cpu().numpy()
    cn, nn = codes.cpu().numpy(), norms.cpu().numpy()
    written = np.zeros((slots, cap), dtype=bool)
    for t in range(steps):
        for r in range(slots):
            if 0 <= pos[t, r] < cap:
                written[r, pos[t, r]] = True
                assert np.array_equal(cn[r, pos[t, r]], cq[r, t]) and nn[r, pos[t, r]] == nq[r, t]
    assert np.all(cn[~written] == 0xAB) and np.all(nn[~written] == -7.0)


def test_append_sets_finer_than_256_rows_and_consumer():
    """set_rows = 1 (one set per slot, any cap): append works, the batch
    kernels refuse the handle, and the decode consumer reads the appended
    cache with head h's set (h % n_sets) against the oracle."""
    d, bits, slots, cap, steps = 128, 3, 6, 40, 40
    p = iq.iq_make_params_sets(d, bits, iq.FULL, SEED, slots, 1, device=0)
    X = iqsynth.unit_vectors(slots * steps, d, 8, np.float16).reshape(slots, steps, d)
    codes, norms = _decode_steps(p, X, cap, steps, iq.F16)
    with pytest.raises(iq.IQError) as e:
        iq.iq_quantize(p, torch.from_numpy(X.reshape(-1, d)).cuda())
    assert e.value.status == 2                     # IQ_ERR_UNSUPPORTED
    q = torch.randn((slots, 4, d), dtype=torch.float16, device="cuda")
    sc = iq.iq_attention_scores(p, codes, norms, q)
    torch.cuda.synchronize()
    cn, nn = codes.cpu().numpy(), norms.cpu().numpy()
    for h in range(slots):
        po = O.make_params(d, bits, iq.FULL, SEED + h)
        Qf = q[h].float().cpu().numpy().astype(np.float64)
        want = A.attention_scores(Qf, O.unpack_codes(cn[h], bits, d), nn[h].astype(np.float64), po)
        tol = 2e-3 * np.linalg.norm(Qf, axis=1)[:, None] * nn[h][None, :]
        assert np.all(np.abs(sc[h].cpu().numpy() - want) <= tol + 1e-30)


def test_append_errors():
    p = iq.iq_make_params(128, 3, iq.FAST, SEED, device=0)
    x = torch.zeros((4, 128), dtype=torch.float16, device="cuda")
    codes = torch.zeros((4, 8, 48), dtype=torch.uint8, device="cuda")
    norms = torch.zeros((4, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(iq.IQError) as e:
        iq.iq_append_kv(p, x, codes, norms, position=8)          # outside [0, cap)
    assert e.value.status == 1
    with pytest.raises(ValueError):
        iq.iq_append_kv(p, x, codes[:3], norms[:3], position=0)   # slot count mismatch
    iq.iq_append_kv(p, x[:0], codes[:0], norms[:0], position=0)   # n_rows = 0: no-op
    raw = torch.zeros(4 * 128 + 8, dtype=torch.float16, device="cuda")
    with pytest.raises(iq.IQError) as e:
        iq.iq_append_kv(p, raw[1:1 + 4 * 128].view(4, 128), codes, norms, position=0)
    assert e.value.status == 3                                     # IQ_ERR_MISALIGNED
