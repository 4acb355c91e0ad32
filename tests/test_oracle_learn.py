"""Oracle pins for learning the rotations (oracle/learn_oracle.py, R29/R30):
central finite differences of the distortion in the free parameters u and in
the block operators M, Fast = Full with q_R = 1, the matrix and quaternion
statements of the gradient against each other, and a descent step.  The C++
chain rule (iq_rot_grad_from_operator_grad) and explicit parameters
(iq_make_params_explicit) are checked here too (host-only handles).  CPU only."""
import numpy as np
import pytest

import iqsynth
from oracle import iq_oracle as O
from oracle import learn_oracle as Lo

SEED = iqsynth.PARAMS_SEED


def _data(n, d, seed=3):
    X = iqsynth.outlier_vectors(n, d, seed, np.float64)
    return X


def _safe_step(X, p, rot, direction, h):
    """L at rot +- h*direction, asserting no quantization decision changes
    (L is smooth between decisions)."""
    out = []
    codes = None
    for sgn in (+1, -1):
        q = Lo.params_from_rot(p.d, p.bits, p.variant, rot + sgn * h * direction)
        c, _, _ = O.encode(X, q)
        if codes is None:
            codes = c
        elif not np.array_equal(codes, c):
            return None
        out.append(Lo.distortion(X, q))
    return (out[0] - out[1]) / (2 * h)


@pytest.mark.parametrize("variant", [O.FULL, O.FAST, O.PLANAR2D])
def test_rot_grad_matches_finite_differences(variant):
    d, bits = 16, 2
    p = O.make_params(d, bits, variant, SEED)
    X = _data(6, d)
    rot = Lo.rot_of(p)
    g = Lo.rot_grad(X, p)
    rng = np.random.default_rng(1)
    checked = 0
    for _ in range(20):
        dirn = rng.standard_normal(rot.size)
        fd = _safe_step(X, p, rot, dirn, 1e-7)
        if fd is None:
            continue
        # the normalisation q = u/||u|| makes the derivative along dirn equal
        # to the projected gradient dotted with dirn (at ||u|| = 1)
        assert fd == pytest.approx(float(g @ dirn), rel=1e-5, abs=1e-9)
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("variant", [O.FULL, O.FAST, O.PLANAR2D])
def test_operator_grad_matches_finite_differences(variant):
    """Perturb one block operator entry directly (M free, not orthogonal)."""
    d, bits = 8, 3
    p = O.make_params(d, bits, variant, SEED)
    X = _data(5, d, seed=7)
    G = Lo.operator_grad(X, p)
    xb, _, _ = Lo._blocks(X, p)
    w = O.block_width(variant)
    # matrix form of the forward map, evaluated by explicit products
    M = np.stack([O.forward_blocks(variant, p.qL[b:b + 1] if p.qL is not None else None,
                                   p.qR[b:b + 1] if p.qR is not None else None,
                                   p.cs[b:b + 1] if p.cs is not None else None,
                                   np.eye(w)[:, None, :]).reshape(w, w).T for b in range(xb.shape[1])])

    def L_of(Mx):
        y = np.einsum("gij,ngj->ngi", Mx, xb).reshape(X.shape[0], -1)
        c = O.dequantize_codes(O.quantize_codes(y, p.cb), p.cb)
        return float(np.sum((y - c) ** 2)), O.quantize_codes(y, p.cb)

    base, codes0 = L_of(M)
    assert base == pytest.approx(Lo.distortion(X, p), rel=1e-12)
    h = 1e-7
    for (b, i, j) in [(0, 0, 0), (1, w - 1, 0), (0, 1, w - 1)]:
        Mp, Mm = M.copy(), M.copy()
        Mp[b, i, j] += h
        Mm[b, i, j] -= h
        (lp, cp), (lm, cm) = L_of(Mp), L_of(Mm)
        if np.array_equal(cp, codes0) and np.array_equal(cm, codes0):
            assert (lp - lm) / (2 * h) == pytest.approx(G[b, i, j], rel=1e-5, abs=1e-9)


def test_fast_equals_full_with_unit_right_factor():
    d, bits = 16, 3
    pf = O.make_params(d, bits, O.FAST, SEED)
    pF = O.make_params(d, bits, O.FULL, SEED)
    pF.qR = np.tile([1.0, 0.0, 0.0, 0.0], (pF.qL.shape[0], 1))
    pF.qL = pf.qL.copy()
    X = _data(20, d)
    gF = Lo.rot_grad(X, pF).reshape(-1, 8)[:, :4]
    assert np.allclose(gF, Lo.rot_grad(X, pf).reshape(-1, 4), rtol=1e-12, atol=1e-14)


def test_descent_step_lowers_distortion():
    d, bits = 32, 2
    p = O.make_params(d, bits, O.FULL, SEED)
    X = _data(400, d, seed=11)
    L0 = Lo.distortion(X, p)
    g = Lo.rot_grad(X, p)
    q = Lo.params_from_rot(d, bits, O.FULL, Lo.rot_of(p) - 1e-3 * g / np.linalg.norm(g))
    assert Lo.distortion(X, q) < L0


def test_cpp_chain_rule_and_explicit_params():
    from __graft_entry__ import load_builder
    load_builder().build()
    import paper_2603_28430_b200 as iq
    d, bits = 16, 3
    for variant in (O.FULL, O.FAST, O.PLANAR2D):
        ph = iq.iq_make_params(d, bits, variant, SEED, device=-1)
        rot = iq.iq_export_params(ph)["rot"]
        # explicit parameters: a scaled copy renormalises to the same handle
        pe = iq.iq_make_params_explicit(d, bits, variant, rot * 3.0, device=-1)
        assert np.allclose(iq.iq_export_params(pe)["rot"], rot, rtol=0, atol=1e-15)
        # chain rule from the oracle's operator gradient equals the oracle's
        # direct quaternion gradient
        po = Lo.params_from_rot(d, bits, variant, rot)
        X = _data(10, d, seed=variant + 5)
        G = Lo.operator_grad(X, po).reshape(-1)
        assert np.allclose(iq.iq_rot_grad_from_operator_grad(ph, G), Lo.rot_grad(X, po), rtol=1e-9, atol=1e-12)
