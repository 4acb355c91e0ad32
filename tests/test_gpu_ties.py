"""Exact fp32 ties and the odd symmetry of the kernels' quantizer (DESIGN.md
R3, R14b; PAPER.md:182 says only "nearest centroid").

Ties.  With explicit parameters whose block operator is L(q) (Fast, or Full
with q_R = 1) the one-hot row e_{4k} rotates to y = q_k exactly: column 0 of
L(q) is q, and the kernel's FMA chain against zeros is exact.  Choosing
quaternion components equal to +-tau_i (the fp32 thresholds the kernels
compare with) puts rotated coordinates EXACTLY on a threshold in the kernel's
arithmetic (rho = 1 exactly, r * tau_i = tau_i).  The kernels' documented rule
(the odd quantizer): |y| >= tau_i counts, so +tau_i codes h + i and -tau_i
codes h - 1 - i (the larger-magnitude centroid on both sides), the other
blocks' +0 coordinates code h.  The oracle decides in fp64 against the exact
midpoints (ties up), so these coordinates sit within ~1e-9 of its thresholds:
inside the parity bar's 1e-5 band, which the oracle check must accept.

Oddness.  The kernels' Q is odd and T is linear with symmetric rounding, so
x^(-x) = -x^(x) bit for bit, codes(-x) = L - 1 - codes(x) and the norms agree."""
import numpy as np
import pytest

import iqsynth
import iq_parity as parity
from oracle import iq_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_28430_b200 as iq  # noqa: E402

NP = {iq.F32: np.float32, iq.F16: np.float16}


def _tie_case(variant, d, bits):
    """(explicit rot, X one-hot rows, expected kernel codes [n, d])."""
    cb = O.make_codebook(d, bits)
    L, h = 1 << bits, 1 << (bits - 1)
    tau = cb.thresholds.astype(np.float32).astype(np.float64)[h:]        # tau_1 < ... < tau_{h-1}
    assert tau.size == h - 1
    w = 2 if variant == iq.PLANAR2D else 4
    g = d // w
    rot, want = [], np.full((g, d), h, dtype=np.int64)                  # +0 coordinates code h
    for k in range(g):
        i, j = 1 + k % (h - 1), 1 + (k + 1) % (h - 1)
        s1, s2 = (-1.0) ** k, (-1.0) ** (k // 2)
        if variant == iq.PLANAR2D:
            s = s1 * tau[i - 1]
            rot += [np.sqrt(1.0 - s * s), s]                              # R(theta) e_0 = (cos, sin)
            comps = {1: (s, i)}
        else:
            b, c = s1 * tau[i - 1], s2 * tau[j - 1]
            a = np.sqrt(0.6 * (1.0 - b * b - c * c))
            q = [a, b, c, np.sqrt(1.0 - a * a - b * b - c * c)]          # unit: a^2+b^2+c^2+d^2 = 1
            rot += q + ([1.0, 0.0, 0.0, 0.0] if variant == iq.FULL else [])
            comps = {1: (b, i), 2: (c, j)}
        for comp, (val, m) in comps.items():
            want[k, w * k + comp] = h + m if val > 0 else h - 1 - m
        want[k, w * k] = -1                                              # not a tie: not asserted
        if variant != iq.PLANAR2D:
            want[k, w * k + 3] = -1
    X = np.zeros((g, d))
    for k in range(g):
        X[k, w * k] = 1.0
    return np.array(rot), X, want


@pytest.mark.parametrize("dt", [iq.F32, iq.F16])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d", [64, 128, 512])
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_exact_fp32_ties_follow_the_odd_rule(variant, dt, d, bits):
    rot, X, want = _tie_case(variant, d, bits)
    p = iq.iq_make_params_explicit(d, bits, variant, rot, device=0)
    ex = iq.iq_export_params(p)
    x = torch.from_numpy(X.astype(NP[dt])).cuda()
    y, codes, norms = iq.iq_roundtrip(p, x, emit_codes=True)
    y1 = iq.iq_roundtrip(p, x)
    cq, nq = iq.iq_quantize(p, x)
    torch.cuda.synchronize()
    assert torch.equal(codes, cq) and torch.equal(norms, nq)
    assert torch.all(norms == 1.0)                                       # rho exact: the ties are exact
    got = O.unpack_codes(codes.cpu().numpy(), bits, d)
    sel = want >= 0
    assert np.array_equal(got[sel], want[sel])
    # the value-only fused kernel builds its output from the same decisions
    po = O.make_params(d, bits, variant, 0)
    po.qL, po.qR, po.cs = _oracle_rot(variant, d, ex["rot"])
    imp, resid = parity.implied_codes(y1.cpu().numpy().astype(np.float64), np.ones(X.shape[0]), po)
    assert resid <= 0.25 and np.array_equal(imp[sel], want[sel])
    # and the oracle's fp64 ties-up decision accepts all of it (boundary band)
    Xs = X.astype(NP[dt])
    _band_only(parity.check(Xs, po, y.cpu().numpy(), codes.cpu().numpy(), norms.cpu().numpy(), NP[dt]), NP[dt])
    rv, resid, zero_ok = parity.check_values(Xs, po, y1.cpu().numpy(), NP[dt])
    assert zero_ok and resid <= 0.25
    _band_only(rv, NP[dt])


def _band_only(r, dt):
    """Tie rows disagree with the oracle only inside the 1e-5 band (the
    agreement fraction is not meaningful on a handful of rows made of ties)."""
    assert r.max_boundary_dist <= parity.BOUNDARY, r
    assert r.max_recon_rel_all <= parity.RECON_RTOL[dt], r
    assert r.max_norm_rel <= parity.NORM_RTOL, r


def _oracle_rot(variant, d, rot):
    """The oracle's parameter arrays from the exported fp64 rotations."""
    if variant == iq.PLANAR2D:
        return None, None, rot.reshape(-1, 2)
    if variant == iq.FULL:
        r = rot.reshape(-1, 8)
        return r[:, :4].copy(), r[:, 4:].copy(), None
    return rot.reshape(-1, 4).copy(), None, None


@pytest.mark.parametrize("dt", [iq.F32, iq.F16])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d,bits", [(128, 3), (128, 4), (512, 2), (256, 4), (64, 1)])
def test_kernels_are_odd(variant, dt, d, bits):
    X = iqsynth.unit_vectors(3000, d, 31 + d + bits, NP[dt])
    p = iq.iq_make_params(d, bits, variant, iqsynth.PARAMS_SEED, device=0)
    xp = torch.from_numpy(X).cuda()
    xn = -xp
    yp, cp, npos = iq.iq_roundtrip(p, xp, emit_codes=True)
    yn, cn, nneg = iq.iq_roundtrip(p, xn, emit_codes=True)
    vp, vn = iq.iq_roundtrip(p, xp), iq.iq_roundtrip(p, xn)
    dp = iq.iq_dequantize(p, cp, npos, dtype=xp.dtype)
    dn = iq.iq_dequantize(p, cn, nneg, dtype=xp.dtype)
    torch.cuda.synchronize()
    assert torch.equal(npos, nneg)
    assert torch.equal(yn, -yp) and torch.equal(vn, -vp) and torch.equal(dn, -dp)
    L = 1 << bits
    a = O.unpack_codes(cp.cpu().numpy(), bits, d)
    b = O.unpack_codes(cn.cpu().numpy(), bits, d)
    assert np.array_equal(a + b, np.full_like(a, L - 1))
