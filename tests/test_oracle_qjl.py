"""Oracle pins for the stage-2 residual sketch (oracle/qjl_oracle.py,
DESIGN.md R20-R24; PAPER.md:355-362 names the construction, QJL defines it).
Each test checks the oracle against something other than itself: the
normal law, brute-force loops, closed-form expectations of the estimator,
special cases.  CPU only."""
import math

import numpy as np
import pytest
from scipy import stats

import iqsynth
from oracle import iq_oracle as O
from oracle import qjl_oracle as Q

SEED = iqsynth.PARAMS_SEED


@pytest.fixture(scope="module")
def S128():
    return Q.sketch_matrix(128, SEED)


def test_sketch_is_standard_normal_in_fp16(S128):
    """R20: i.i.d. N(0,1) entries, each an IEEE half value."""
    v = S128.ravel()
    assert np.array_equal(v, v.astype(np.float16).astype(np.float64))
    ks = stats.kstest(v, "norm")
    assert ks.pvalue > 1e-3, ks
    assert abs(v.mean()) < 4 / math.sqrt(v.size)
    assert abs(v.var() - 1.0) < 4 * math.sqrt(2 / v.size)
    # rows are uncorrelated (a transposed or repeated stream would not be)
    c = np.corrcoef(S128[:64])
    off = c[~np.eye(64, dtype=bool)]
    assert np.abs(off).max() < 0.4 and abs(off.mean()) < 0.01


def test_sketch_depends_on_seed_and_key():
    a = Q.sketch_matrix(16, 1)
    b = Q.sketch_matrix(16, 2)
    assert not np.array_equal(a, b)
    # keyed stream: differs from the rotation stream of the same seed
    g = np.array([O.gaussian(1, j) for j in range(16 * 16)]).astype(np.float16).astype(np.float64)
    assert not np.array_equal(a.ravel(), g)


def test_bits_by_brute_force_loops():
    d = 8
    S = Q.sketch_matrix(d, 7)
    rng = np.random.default_rng(3)
    R = rng.standard_normal((5, d))
    bits = Q.sketch_bits(R, S)
    for r in range(5):
        for i in range(d):
            z = 0.0
            for k in range(d):
                z += S[i, k] * R[r, k]
            assert bits[r, i] == (1 if z >= 0 else 0)


def test_one_hot_residual_gives_column_signs(S128):
    for k in (0, 17, 127):
        r = np.zeros((1, 128))
        r[0, k] = 0.25
        assert np.array_equal(Q.sketch_bits(r, S128)[0], (S128[:, k] >= 0).astype(np.uint8))
        r[0, k] = -0.25
        assert np.array_equal(Q.sketch_bits(r, S128)[0], (S128[:, k] <= 0).astype(np.uint8) | (S128[:, k] == 0))


def test_zero_residual():
    """x = 0: x^ = 0 (Alg.1 with rho = 0), r = 0, gamma = 0, z = 0 -> q = +1."""
    p = O.make_params(64, 3, O.FULL, SEED)
    S = Q.sketch_matrix(64, SEED)
    codes, packed, rho, xh, q, g = Q.encode(np.zeros((2, 64)), p, S)
    assert np.all(g == 0) and np.all(q == 1) and np.all(xh == 0)
    assert np.array_equal(Q.correction(q, g, S), np.zeros((2, 64)))


def test_pack_bits_lsb_first():
    q = np.zeros((1, 16), dtype=np.uint8)
    q[0, 0] = 1
    q[0, 9] = 1
    q[0, 15] = 1
    assert Q.pack_bits(q).tolist() == [[0x01, 0x82]]
    rng = np.random.default_rng(0)
    q = rng.integers(0, 2, (3, 128)).astype(np.uint8)
    assert np.array_equal(Q.unpack_bits(Q.pack_bits(q), 128), q)


def test_sign_correlation_closed_form():
    """E_s[(s.y) sign(s.r)] = sqrt(2/pi) <y, r> / ||r|| for s ~ N(0, I):
    the identity the sqrt(pi/2) factor of R24 inverts.  Rows of sketches of
    many seeds are the samples."""
    d = 32
    rng = np.random.default_rng(11)
    y, r = rng.standard_normal(d), rng.standard_normal(d)
    rows = np.vstack([Q.sketch_matrix(d, 1000 + s) for s in range(120)])   # 3840 samples
    samples = (rows @ y) * np.where(rows @ r >= 0, 1.0, -1.0)
    want = math.sqrt(2 / math.pi) * float(y @ r) / float(np.linalg.norm(r))
    se = samples.std() / math.sqrt(samples.size)
    assert abs(samples.mean() - want) < 4 * se + 1e-3 * abs(want), (samples.mean(), want, se)


def test_inner_product_estimator_unbiased_and_variance_bound():
    """R24 over independent sketches: mean of the estimate of <y, x> equals
    <y, x>; its variance obeys the QJL bound (pi/2 - 1 + 1)/m ||y||^2 ||r||^2
    (a per-sample second moment of pi/2 ||y||^2 ||r||^2 / m at most)."""
    d, bits = 32, 2
    p = O.make_params(d, bits, O.FULL, SEED)
    rng = np.random.default_rng(5)
    X = rng.standard_normal((1, d))
    Y = rng.standard_normal((1, d))
    est = []
    for s in range(150):
        S = Q.sketch_matrix(d, 2000 + s)
        codes, packed, rho, xh, q, g = Q.encode(X, p, S)
        est.append(Q.inner_product(Y, xh, q, g, S)[0])
    est = np.array(est)
    truth = float(X[0] @ Y[0])
    r = X[0] - xh[0]
    bound = (math.pi / 2) / d * float(Y[0] @ Y[0]) * float(r @ r)
    assert est.var() <= 1.5 * bound
    assert abs(est.mean() - truth) < 4 * math.sqrt(bound / est.size), (est.mean(), truth)
    # and the stage-1 estimate alone is biased by <y, r> (what stage 2 corrects)
    assert abs(float(Y[0] @ xh[0]) - truth) == pytest.approx(abs(float(Y[0] @ r)), rel=1e-12)


def test_reconstruction_unbiased():
    """E_S[x~] = x for x~ = x^ + sqrt(pi/2)/m gamma S^T q (R24)."""
    d = 16
    p = O.make_params(d, 2, O.FAST, SEED)
    X = np.random.default_rng(9).standard_normal((1, d))
    acc = np.zeros(d)
    N = 300
    for s in range(N):
        S = Q.sketch_matrix(d, 5000 + s)
        codes, packed, rho, xh, q, g = Q.encode(X, p, S)
        acc += (xh + Q.correction(q, g, S))[0]
    mean = acc / N
    r = X[0] - xh[0]
    # per-coordinate std of one sample <= sqrt(pi/2) ||r|| (1 + ...)/sqrt(m)
    tol = 4 * math.sqrt(math.pi / 2) * float(np.linalg.norm(r)) / math.sqrt(N)
    assert np.abs(mean - X[0]).max() < tol, (np.abs(mean - X[0]).max(), tol)


def test_gamma_is_residual_norm_and_scale_equivariance(S128):
    p = O.make_params(128, 3, O.FULL, SEED)
    X = iqsynth.unit_vectors(64, 128, 77, np.float32).astype(np.float64)
    c1, _, _, xh1, q1, g1 = Q.encode(X, p, S128)
    c2, _, _, xh2, q2, g2 = Q.encode(4.0 * X, p, S128)      # power of two: exact
    assert np.array_equal(c1, c2) and np.array_equal(q1, q2)
    assert np.allclose(g2, 4.0 * g1, rtol=1e-14)
    assert np.allclose(g1, np.linalg.norm(X - xh1, axis=1), rtol=1e-14)
    # closed form of Appendix A.2: E||r||^2 per unit vector = d * D_f(b)
    want = O.expected_unit_vector_mse(128, 3) * 128
    assert np.mean(g1 ** 2) == pytest.approx(want, rel=0.15)
