"""Oracle pins: RNG, quaternion algebra, the Proposition, block structure,
complexity counts (PAPER.md Sections 4-6, Table 1).  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import iq_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- RNG [R12]
def test_splitmix64_reference_outputs():
    g = _gold("splitmix64.json")
    c0 = g["cases"][0]
    assert [format(O.splitmix64(c0["seed"], k), "016x") for k in range(3)] == c0["outputs_hex"]
    c1 = g["cases"][1]
    assert [str(O.splitmix64(c1["seed"], k)) for k in range(3)] == c1["outputs_dec"]


def test_uniform_range_and_moments():
    u = np.array([O.uniform01(7, k) for k in range(200000)])
    assert u.min() > 0.0 and u.max() <= 1.0
    assert abs(u.mean() - 0.5) < 4 * math.sqrt(1 / 12 / u.size)
    assert stats.kstest(u, "uniform").pvalue > 1e-3


def test_box_muller_is_standard_normal():
    z = np.array([O.gaussian(20260331, j) for j in range(200000)])
    n = z.size
    assert abs(z.mean()) < 5 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2 / n)
    assert abs(np.mean(z ** 4) - 3.0) < 5 * math.sqrt(96 / n)
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_params_deterministic_and_fast_shares_full_qL():
    a = O.make_rotation_params(128, O.FULL, 5)
    b = O.make_rotation_params(128, O.FULL, 5)
    f = O.make_rotation_params(128, O.FAST, 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[0], f[0]) and f[1] is None
    assert not np.array_equal(a[0], O.make_rotation_params(128, O.FULL, 6)[0])


def test_haar_quaternion_moments():
    """Gaussian-normalize sampling on S^3: unit norm, E[q_c]=0,
    E[q_c^2]=1/4 (uniform on S^3)."""
    qL, qR, _ = O.make_rotation_params(4 * 20000, O.FULL, 11)
    q = np.concatenate([qL, qR])
    assert np.max(np.abs(np.linalg.norm(q, axis=1) - 1.0)) < 1e-15 * 4
    n = q.shape[0]
    assert np.all(np.abs(q.mean(axis=0)) < 5 * math.sqrt(0.25 / n))
    assert np.all(np.abs((q * q).mean(axis=0) - 0.25) < 5 * math.sqrt(0.25 * 0.75 / 4 / n) + 2e-3)


def _f4_cdf(z):
    # CDF of f_4(z) = (2/pi) sqrt(1 - z^2), integrated by hand
    return 0.5 + (z * np.sqrt(1 - z * z) + np.arcsin(z)) / np.pi


def _f2_cdf(z):
    # CDF of the arcsine law f_2(z) = 1 / (pi sqrt(1 - z^2))
    return 0.5 + np.arcsin(z) / np.pi


def test_marginal_law_of_random_block_rotation_full_fast():
    """for a fixed block and Haar R_b, each rotated coordinate of a
    unit block has density f_4.  Test the oracle's Full and Fast transforms
    with freshly sampled parameters per block on e_0 and on a generic unit
    block: KS against the closed-form CDF of f_4; second moment r^2/k."""
    g = 40000
    for variant in (O.FULL, O.FAST):
        qL, qR, _ = O.make_rotation_params(4 * g, variant, 3 + variant)
        for x in (np.array([1.0, 0, 0, 0]), np.array([0.5, -0.1, 0.7, 0.2])):
            x = x / np.linalg.norm(x)
            y = O.forward_blocks(variant, qL, qR, None, np.tile(x, (g, 1)))
            for j in range(4):
                assert stats.kstest(y[:, j], _f4_cdf).pvalue > 1e-4
                assert abs(np.mean(y[:, j] ** 2) - 0.25) < 5 * math.sqrt(1 / 8 / g)
            assert abs(np.mean(y[:, 0] ** 4) - 1 / 8) < 0.01  # int z^4 f_4 = 1/8


def test_marginal_law_planar_is_arcsine():
    _, _, cs = O.make_rotation_params(2 * 50000, O.PLANAR2D, 9)
    u = O.forward_blocks(O.PLANAR2D, None, None, cs, np.tile([1.0, 0.0], (cs.shape[0], 1)))
    assert stats.kstest(u[:, 0], _f2_cdf).pvalue > 1e-4
    assert stats.kstest(u[:, 1], _f2_cdf).pvalue > 1e-4
    assert abs(np.mean(u[:, 0] ** 2) - 0.5) < 0.01


def test_marginal_pdf_normalisation():
    assert O.sphere_marginal_pdf(4, 0.0) == pytest.approx(2 / math.pi, abs=1e-14)
    assert O.sphere_marginal_pdf(2, 0.0) == pytest.approx(1 / math.pi, abs=1e-14)
    assert O.sphere_marginal_pdf(4, 1.0) == 0.0
    from scipy.integrate import quad
    for k in (3, 4, 8, 128):
        val, _ = quad(lambda z: float(O.sphere_marginal_pdf(k, z)), -1, 1)
        assert val == pytest.approx(1.0, abs=1e-8)


# ------------------------------------------------------ quaternions
E = [np.eye(4)[i] for i in range(4)]   # 1, i, j, k


def test_defining_relations():
    one, i, j, k = E
    for u in (i, j, k):
        assert np.array_equal(O.qmul(u, u), -one)                    # i^2=j^2=k^2=-1
    assert np.array_equal(O.qmul(O.qmul(i, j), k), -one)             # ijk = -1
    # consequences of the relations (Hamilton): ij=k, jk=i, ki=j, ji=-k
    assert np.array_equal(O.qmul(i, j), k)
    assert np.array_equal(O.qmul(j, k), i)
    assert np.array_equal(O.qmul(k, i), j)
    assert np.array_equal(O.qmul(j, i), -k)
    for u in E:
        assert np.array_equal(O.qmul(one, u), u) and np.array_equal(O.qmul(u, one), u)


def test_bilinear_expansion_on_basis():
    """qmul(a,b) == sum_mn a_m b_n e_m e_n with the basis table fixed by the
    defining relations (catches any sign/index error in the 16-term formula)."""
    rng = np.random.default_rng(0)
    table = {}
    one, i, j, k = E
    # basis products derived from i^2=j^2=k^2=ijk=-1
    rel = {(0, 0): one, (0, 1): i, (0, 2): j, (0, 3): k,
           (1, 0): i, (1, 1): -one, (1, 2): k, (1, 3): -j,
           (2, 0): j, (2, 1): -k, (2, 2): -one, (2, 3): i,
           (3, 0): k, (3, 1): j, (3, 2): -i, (3, 3): -one}
    table.update(rel)
    for _ in range(50):
        a, b = rng.standard_normal(4), rng.standard_normal(4)
        ref = sum(a[m] * b[n] * table[(m, n)] for m in range(4) for n in range(4))
        assert np.allclose(O.qmul(a, b), ref, atol=1e-14)


def test_worked_examples_and_conjugate():
    g = _gold("spec_worked_examples.json")
    for c in g["qmul"]:
        assert np.array_equal(O.qmul(np.array(c["a"], float), np.array(c["b"], float)), np.array(c["out"], float))
    q = np.array([1.0, 2, 3, 4])
    assert np.array_equal(O.qmul(q, O.qconj(q)), np.array([30.0, 0, 0, 0]))
    assert np.array_equal(O.qconj(q), np.array([1.0, -2, -3, -4]))


def test_norm_multiplicative_and_associative():
    rng = np.random.default_rng(1)
    a, b, c = rng.standard_normal((3, 1000, 4))
    assert np.allclose(np.linalg.norm(O.qmul(a, b), axis=1),
                       np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1), rtol=1e-12)
    assert np.allclose(O.qmul(O.qmul(a, b), c), O.qmul(a, O.qmul(b, c)), atol=1e-12)


# --------------------------------------------- Proposition
def _block_matrix(variant, qL, qR):
    return np.stack([O.forward_blocks(variant, qL, qR, None, e) for e in E], axis=-1)


def test_proposition_orthogonal_inverse_doublecover():
    qL, qR, _ = O.make_rotation_params(4 * 500, O.FULL, 21)
    rng = np.random.default_rng(2)
    v = rng.standard_normal((500, 4))
    for variant in (O.FULL, O.FAST):
        t = O.forward_blocks(variant, qL, qR, None, v)
        assert np.allclose(np.linalg.norm(t, axis=1), np.linalg.norm(v, axis=1), rtol=1e-12)
        back = O.inverse_blocks(variant, qL, qR, None, t)
        assert np.max(np.abs(back - v)) < 1e-12
    # (q_L, q_R) and (-q_L, -q_R) induce the same element of SO(4)
    t1 = O.forward_blocks(O.FULL, qL, qR, None, v)
    t2 = O.forward_blocks(O.FULL, -qL, -qR, None, v)
    assert np.max(np.abs(t1 - t2)) < 1e-14
    # explicit 4x4 matrices: orthogonal, det +1
    for variant in (O.FULL, O.FAST):
        M = np.stack([_block_matrix(variant, qL[b], None if qR is None else qR[b]) for b in range(50)])
        assert np.allclose(np.einsum("bij,bkj->bik", M, M), np.eye(4), atol=1e-13)
        assert np.allclose(np.linalg.det(M), 1.0, atol=1e-12)


def test_full_with_unit_qR_equals_fast_bitwise():
    qL, _, _ = O.make_rotation_params(64, O.FAST, 4)
    one = np.tile([1.0, 0, 0, 0], (qL.shape[0], 1))
    v = np.random.default_rng(3).standard_normal((qL.shape[0], 4))
    full = O.forward_blocks(O.FULL, qL, one, None, v)
    fast = O.forward_blocks(O.FAST, qL, None, None, v)
    assert np.array_equal(full, fast)
    assert np.array_equal(O.inverse_blocks(O.FULL, qL, one, None, v), O.inverse_blocks(O.FAST, qL, None, None, v))


def test_commuting_isoclinic_factors():
    """sandwich(q_L,1) o sandwich(1,q_R) == sandwich(q_L,q_R)."""
    qL, qR, _ = O.make_rotation_params(4 * 100, O.FULL, 8)
    one = np.tile([1.0, 0, 0, 0], (100, 1))
    v = np.random.default_rng(4).standard_normal((100, 4))
    a = O.forward_blocks(O.FULL, qL, one, None, O.forward_blocks(O.FULL, one, qR, None, v))
    b = O.forward_blocks(O.FULL, one, qR, None, O.forward_blocks(O.FULL, qL, one, None, v))
    c = O.forward_blocks(O.FULL, qL, qR, None, v)
    assert np.allclose(a, c, atol=1e-14) and np.allclose(b, c, atol=1e-14)


def test_left_multiplication_by_i():
    i = np.array([[0.0, 1, 0, 0]])
    one = np.array([[1.0, 0, 0, 0]])
    assert np.array_equal(O.forward_blocks(O.FULL, i, one, None, one), i)


def test_planar_quarter_turn():
    cs = np.array([[math.cos(math.pi / 2), math.sin(math.pi / 2)]])
    f = O.forward_blocks(O.PLANAR2D, None, None, cs, np.array([[1.0, 0.0]]))
    assert np.allclose(f, [[0.0, 1.0]], atol=1e-16)
    assert np.allclose(O.inverse_blocks(O.PLANAR2D, None, None, cs, f), [[1.0, 0.0]], atol=1e-16)


# ----------------------------------------- block structure
def test_block_count_and_locality():
    g = _gold("paper_table1.json")["d128"]
    for name, variant in (("full", O.FULL), ("fast", O.FAST), ("planar2d", O.PLANAR2D)):
        p = O.make_params(128, 2, variant, 1)
        n_blocks = (p.qL.shape[0] if variant != O.PLANAR2D else p.cs.shape[0])
        assert n_blocks == g[name]["blocks"]
    p = O.make_params(128, 3, O.FULL, 1)
    x = np.random.default_rng(5).standard_normal((1, 128))
    x2 = x.copy()
    x2[0, 8:12] += 0.3            # perturb block 2 only
    y0 = O.rotated_coordinates(x, p)[0] * np.linalg.norm(x)
    y2 = O.rotated_coordinates(x2, p)[0] * np.linalg.norm(x2)
    others = np.setdiff1d(np.arange(128), np.arange(8, 12))
    assert np.allclose(y2[others], y0[others], atol=1e-13)      # untouched blocks
    assert np.all(np.abs(y2[8:12] - y0[8:12]) > 1e-6)            # block 2 moved


def test_block_diagonal_matrix_oracle_small_d():
    """For d <= 16 the blockwise map equals the assembled block-diagonal
    element of (SO(4))^g."""
    for variant in (O.FULL, O.FAST, O.PLANAR2D):
        p = O.make_params(16, 2, variant, 13)
        w = O.block_width(variant)
        Mfull = np.zeros((16, 16))
        for b in range(16 // w):
            for c in range(w):
                e = np.zeros((1, 1, w)); e[0, 0, c] = 1.0
                if variant == O.PLANAR2D:
                    col = O.forward_blocks(variant, None, None, p.cs[b:b + 1], e)
                else:
                    col = O.forward_blocks(variant, p.qL[b:b + 1], None if p.qR is None else p.qR[b:b + 1], None, e)
                Mfull[b * w:(b + 1) * w, b * w + c] = col.reshape(-1)
        assert np.allclose(Mfull @ Mfull.T, np.eye(16), atol=1e-13)
        x = np.random.default_rng(6).standard_normal((3, 16))
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        assert np.allclose(O.rotated_coordinates(x, p), x @ Mfull.T, atol=1e-14)


# ------------------------------------------------ complexity (Table 1)
def test_table1_counts_at_d128():
    g = _gold("paper_table1.json")["d128"]
    for name, variant in (("full", O.FULL), ("fast", O.FAST), ("planar2d", O.PLANAR2D)):
        params, fmas = O.complexity(variant, 128)
        assert (params, fmas) == (g[name]["params"], g[name]["fmas"]), name


@pytest.mark.parametrize("d", [64, 256, 512, 100])
def test_general_formulas_p333(d):
    g4, g2 = -(-d // 4), -(-d // 2)
    assert O.complexity(O.FULL, d) == (8 * g4, 32 * g4)
    assert O.complexity(O.FAST, d) == (4 * g4, 16 * g4)
    assert O.complexity(O.PLANAR2D, d) == (2 * g2, 4 * g2)
