"""Oracle pins for the decode consumer (oracle/attn_oracle.py, R25-R27):
brute-force loops, the rotation duality <q, T^-1 c> = <T q, c> the kernel
relies on (computed here with the oracle's forward transform, a different
formula), and consistency of the two-stage logit with the pinned QJL
estimator.  CPU only."""
import numpy as np
import pytest

import iqsynth
from oracle import attn_oracle as A
from oracle import iq_oracle as O
from oracle import qjl_oracle as Q

SEED = iqsynth.PARAMS_SEED


def _keys(n, d, bits, variant, seed=3):
    p = O.make_params(d, bits, variant, SEED)
    X = iqsynth.unit_vectors(n, d, seed, np.float32).astype(np.float64) * 1.7
    codes, packed, rho = O.encode(X, p)
    return p, X, codes, rho


@pytest.mark.parametrize("variant", [O.FULL, O.FAST, O.PLANAR2D])
def test_brute_force_loops(variant):
    d = 8
    p, X, codes, rho = _keys(5, d, 3, variant)
    Qm = np.random.default_rng(1).standard_normal((3, d))
    s = A.attention_scores(Qm, codes, rho, p)
    xh = O.decode(codes, rho, p)
    for j in range(3):
        for k in range(5):
            acc = 0.0
            for i in range(d):
                acc += Qm[j, i] * xh[k, i]
            assert s[j, k] == pytest.approx(acc, rel=1e-13, abs=1e-15)


@pytest.mark.parametrize("variant", [O.FULL, O.FAST, O.PLANAR2D])
def test_rotation_duality(variant):
    """<q, rho T^-1(C[code])> = rho <T q, C[code]> (T orthogonal)."""
    d = 64
    p, X, codes, rho = _keys(40, d, 3, variant)
    Qm = np.random.default_rng(2).standard_normal((4, d))
    s = A.attention_scores(Qm, codes, rho, p)
    w = O.block_width(variant)
    Tq = O.forward_blocks(variant, p.qL, p.qR, p.cs, Qm.reshape(4, -1, w)).reshape(4, -1)
    c = O.dequantize_codes(codes, p.cb)
    s2 = (Tq @ c.T) * rho[None, :]
    assert np.allclose(s, s2, rtol=1e-12, atol=1e-12)


def test_two_stage_matches_qjl_estimator():
    d = 32
    p, X, codes, rho = _keys(16, d, 2, O.FULL)
    S = Q.sketch_matrix(d, SEED)
    _, _, _, xh, q01, g = Q.encode(X, p, S)
    Y = np.random.default_rng(4).standard_normal((16, d))
    s = A.attention_scores(Y, codes, rho, p, q01, g, S)
    est = Q.inner_product(Y, xh, q01, g, S)            # row-wise <y_i, x_i>
    assert np.allclose(np.diag(s), est, rtol=1e-12, atol=1e-12)


def test_stage_two_reduces_logit_error_on_average():
    """The complete two-stage estimate is unbiased; over many keys its mean
    error is far below the stage-1 bias magnitude for a query aligned with
    the residuals (PAPER.md:460's quantity)."""
    d = 64
    p, X, codes, rho = _keys(2000, d, 2, O.FULL, seed=9)
    S = Q.sketch_matrix(d, SEED)
    _, _, _, xh, q01, g = Q.encode(X, p, S)
    R = X - xh
    q = R.mean(axis=0, keepdims=True) * 50 + np.random.default_rng(0).standard_normal((1, d)) * 0.01
    truth = (q @ X.T)[0]
    s1 = A.attention_scores(q, codes, rho, p)[0]
    s2 = A.attention_scores(q, codes, rho, p, q01, g, S)[0]
    assert abs(np.mean(s2 - truth)) < 0.25 * abs(np.mean(s1 - truth))
