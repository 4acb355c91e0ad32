"""Oracle pins: Lloyd-Max codebook, nearest-centroid coding, packing, and the
end-to-end Algorithm 1 against closed forms.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.integrate import quad

import iqsynth
from oracle import iq_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------ Lloyd-Max [R1]
def test_one_bit_closed_form():
    lv, dist = O.lloyd_max_gaussian(1)
    assert lv[1] == pytest.approx(math.sqrt(2 / math.pi), abs=1e-14)
    assert lv[0] == -lv[1]
    assert dist == pytest.approx(1 - 2 / math.pi, abs=1e-14)


def test_lloyd_max_matches_max_1960_table():
    g = _gold("lloyd_max_gaussian.json")
    for b in (1, 2, 3, 4):
        lv, dist = O.lloyd_max_gaussian(b)
        pos = lv[len(lv) // 2:]
        assert np.allclose(pos, g["levels_positive"][str(b)], atol=g["tolerance_abs"]), b
        assert dist == pytest.approx(g["distortion"][str(b)], rel=g["distortion_tolerance_rel"]), b


def test_lloyd_conditions_by_quadrature():
    """Centroid condition re-checked by direct numerical integration of
    z * phi(z) over each cell (independent of the closed-form update)."""
    phi = lambda z: math.exp(-0.5 * z * z) / math.sqrt(2 * math.pi)
    for b in (2, 3, 4):
        lv, _ = O.lloyd_max_gaussian(b)
        t = [-np.inf] + [0.5 * (lv[k] + lv[k + 1]) for k in range(len(lv) - 1)] + [np.inf]
        for k in range(len(lv)):
            m0, _ = quad(phi, t[k], t[k + 1], epsabs=1e-14)
            m1, _ = quad(lambda z: z * phi(z), t[k], t[k + 1], epsabs=1e-14)
            assert m1 / m0 == pytest.approx(lv[k], abs=1e-9)


def test_codebook_structure():
    for d in (64, 128, 256, 512):
        for b in (1, 2, 3, 4):
            cb = O.make_codebook(d, b)
            L = 1 << b
            C, T = cb.centroids, cb.thresholds
            assert C.shape == (L,) and T.shape == (L - 1,)
            assert np.array_equal(C, -C[::-1])                        # symmetric [R2]
            assert T[L // 2 - 1] == 0.0                                # middle threshold
            assert np.all(np.diff(C) > 0) and np.all(np.diff(T) > 0)
            assert np.array_equal(C.astype(np.float32).astype(np.float64), C)
            assert np.array_equal(T, -T[::-1])
            # exact fp64 midpoints of the fp32 centroids [R14b]: 2T - C_k is
            # C_{k+1} bit for bit (no rounding anywhere)
            assert T.dtype == np.float64
            assert np.array_equal(2.0 * T - C[:-1], C[1:])
            assert np.array_equal(2.0 * T - C[1:], C[:-1])
            # scaled by 1/sqrt(d): variance-1/d coordinates (P:273 with k=d)
            assert np.allclose(C * math.sqrt(d), cb.levels_unit, rtol=1e-6)


# ------------------------------------------------------------ quantize [R3][R4]
def _custom_codebook(levels):
    C = np.asarray(levels, dtype=np.float32).astype(np.float64)
    T = (C[:-1] + C[1:]) / 2
    return O.Codebook(bits=int(math.log2(len(C))), d=1, centroids=C, thresholds=T, levels_unit=C)


def test_spec_quantizer_examples():
    for c in _gold("spec_worked_examples.json")["quantize"]:
        cb = _custom_codebook(c["levels"])
        assert int(O.quantize_codes(np.array([c["v"]]), cb)[0]) == c["code"]


def test_ties_go_up_and_signed_zero():
    """[R3]: a value exactly on a threshold takes the upper code, at
    negative thresholds too; +-0 code on the positive side; the count clamps
    [R4].  The SPEC's negative-threshold example: levels (-.75,-.25,.25,.75),
    v = -0.5 (the midpoint of -0.75 and -0.25) codes 1."""
    cb = O.make_codebook(128, 3)
    T = cb.thresholds                                                    # t_0..t_6, t_3 = 0
    codes = O.quantize_codes(T, cb)
    assert np.array_equal(codes, [1, 2, 3, 4, 5, 6, 7])                 # t_k -> k+1
    assert O.quantize_codes(np.array([0.0, -0.0]), cb).tolist() == [4, 4]   # +-0 -> upper half
    assert O.quantize_codes(np.array([-1e9, 1e9]), cb).tolist() == [0, 7]   # clamp
    below = np.nextafter(T, -np.inf)                                     # one fp64 ulp below
    assert np.array_equal(O.quantize_codes(below, cb), [0, 1, 2, 3, 4, 5, 6])
    spec = _custom_codebook([-0.75, -0.25, 0.25, 0.75])
    assert O.quantize_codes(np.array([-0.5, 0.5, 0.0]), spec).tolist() == [1, 3, 2]


def test_quantizer_is_odd_off_ties():
    """Q(-y) = -Q(y) for every y that is not a threshold (symmetric codebook
    [R2]); at a nonzero threshold the tie rule breaks the symmetry by one
    level (ties go up on both sides)."""
    rng = np.random.default_rng(11)
    for b in (1, 2, 3, 4):
        cb = O.make_codebook(256, b)
        y = (rng.standard_normal(5000) * 0.08)
        y = y[np.min(np.abs(np.abs(y)[:, None] - cb.thresholds[None, :]), axis=1) > 0]
        qp = O.dequantize_codes(O.quantize_codes(y, cb), cb)
        qn = O.dequantize_codes(O.quantize_codes(-y, cb), cb)
        assert np.array_equal(qn, -qp)
        t = cb.thresholds[cb.thresholds > 0]
        if t.size:
            up, dn = O.quantize_codes(t, cb), O.quantize_codes(-t, cb)
            assert np.array_equal(up + dn, np.full(t.shape, (1 << b)))   # symmetric would give L-1


def test_nearest_centroid_brute_force():
    """code == argmin_k |y - C_k| (ties to the larger k), by brute force over
    all L centroids, on random fp64 values plus values 1e-15 on either side
    of every midpoint (exact midpoints are covered by the tie test; the
    brute-force distances resolve ~1e-17 here)."""
    rng = np.random.default_rng(7)
    for b in (1, 2, 3, 4):
        cb = O.make_codebook(128, b)
        mids = (cb.centroids[:-1] + cb.centroids[1:]) / 2
        y = np.concatenate([rng.standard_normal(20000) * 0.12,
                            mids + 1e-15, mids - 1e-15])
        dist = np.abs(y[:, None] - cb.centroids[None, :])
        L = len(cb.centroids)
        brute = L - 1 - np.argmin(dist[:, ::-1], axis=1)     # ties -> larger k
        assert np.array_equal(O.quantize_codes(y, cb), brute)


# ------------------------------------------------------------ packing [R7]
def test_pack_examples():
    for c in _gold("spec_worked_examples.json")["pack"]:
        out = O.pack_codes(np.array([c["codes"]]), c["bits"])
        if "bytes_hex" in c:
            assert [format(v, "02x") for v in out[0]] == c["bytes_hex"]
        if "nbytes" in c:
            assert out.shape[1] == c["nbytes"]


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 8])
def test_pack_bijection(bits):
    rng = np.random.default_rng(bits)
    codes = rng.integers(0, 1 << bits, size=(37, 61))
    packed = O.pack_codes(codes, bits)
    assert packed.shape[1] == -(-61 * bits // 8)
    assert np.array_equal(O.unpack_codes(packed, bits, 61), codes)


def test_pack_bit_order_independent_formula():
    """Independent restatement: the row bitstream as a big integer equals
    sum_j code_j << (j*b), and bytes are that integer little-endian."""
    rng = np.random.default_rng(3)
    for bits in (2, 3, 4):
        codes = rng.integers(0, 1 << bits, size=(5, 40))
        packed = O.pack_codes(codes, bits)
        for r in range(5):
            v = sum(int(c) << (j * bits) for j, c in enumerate(codes[r]))
            assert v.to_bytes(packed.shape[1], "little") == packed[r].tobytes()


# ------------------------------------------------------------ Algorithm 1
def test_norm_split():
    X = iqsynth.gaussian_rows(50, 128, 1, np.float64, sigma=3.0)
    _, _, rho = O.encode(X, O.make_params(128, 3, O.FULL, 1))
    assert np.allclose(rho, np.linalg.norm(X, axis=1), rtol=1e-15)


def test_zero_vector_gives_exact_zeros():
    for variant in (O.FULL, O.FAST, O.PLANAR2D):
        p = O.make_params(128, 3, variant, 2)
        X = np.zeros((3, 128))
        xh, codes, _, rho = O.roundtrip(X, p)
        assert np.all(xh == 0.0) and np.all(rho == 0.0)
        assert np.all(codes == 4)                            # y = +-0 -> upper half


def test_scale_equivariance():
    """x^(a x) = a x^(x) for a > 0: exactly for powers of two."""
    X = iqsynth.unit_vectors(200, 128, 3, np.float64)
    for variant in (O.FULL, O.FAST, O.PLANAR2D):
        p = O.make_params(128, 3, variant, 3)
        base = O.roundtrip(X, p)[0]
        assert np.array_equal(O.roundtrip(4.0 * X, p)[0], 4.0 * base)
        got = O.roundtrip(3.7 * X, p)[0]
        assert np.allclose(got, 3.7 * base, rtol=1e-12, atol=1e-15)


def test_identity_params_all_variants_agree():
    X = iqsynth.unit_vectors(300, 64, 4, np.float64)
    out = [O.roundtrip(X, O.identity_params(64, 3, v)) for v in (O.FULL, O.FAST, O.PLANAR2D)]
    for o in out[1:]:
        assert np.array_equal(o[1], out[0][1])
    cb = O.make_codebook(64, 3)
    xbar = X / np.linalg.norm(X, axis=1, keepdims=True)
    assert np.array_equal(out[0][1], O.quantize_codes(xbar, cb))


def test_decode_packed_equals_decode():
    X = iqsynth.unit_vectors(100, 128, 5, np.float32)
    p = O.make_params(128, 3, O.FULL, 5)
    xh, codes, packed, rho = O.roundtrip(X, p)
    assert packed.shape == (100, 48)
    assert np.array_equal(O.decode_packed(packed, rho, p), xh)


def test_padding_is_dropped():
    for variant, d in ((O.PLANAR2D, 7), (O.FULL, 6), (O.FAST, 10)):
        p = O.make_params(d, 2, variant, 6)
        X = iqsynth.unit_vectors(10, d, 6, np.float64)
        xh, codes, packed, rho = O.roundtrip(X, p)
        assert xh.shape == (10, d)
        assert packed.shape[1] == O.code_bytes_per_vector(d, 2, variant)


@pytest.mark.parametrize("d", [128, 256, 512])
def test_mse_matches_closed_form_for_every_variant(d):
    """E||xbar - xbar_rec||^2 = d * int (z - Q(z))^2 f_d(z) dz for unit vectors
    uniform on S^{d-1} and ANY fixed orthogonal block rotation (P:277-279
    with k = d).  Monte Carlo within 5 standard errors."""
    n = 6000 if d < 512 else 3000
    X = iqsynth.unit_vectors(n, d, 100 + d, np.float64)
    for b in (2, 3, 4):
        expect = O.expected_unit_vector_mse(d, b)
        for variant in (O.FULL, O.FAST, O.PLANAR2D):
            p = O.make_params(d, b, variant, 20260331)
            xh = O.roundtrip(X, p)[0]
            per_vec = np.mean((X - xh) ** 2, axis=1)
            se = per_vec.std() / math.sqrt(n)
            assert abs(per_vec.mean() - expect) < 5 * se, (d, b, variant)


def test_closed_form_values_survey_appendix():
    """Cross-check two quadrature values against SURVEY.md App. A.2 (computed
    there with the fp64 codebook; ours is the fp32 codebook, so 1e-4 rel)."""
    assert O.expected_unit_vector_mse(128, 3) == pytest.approx(2.654615e-04, rel=1e-4)
    assert O.expected_unit_vector_mse(256, 2) == pytest.approx(4.560207e-04, rel=1e-4)


def test_mse_monotone_in_bits():
    X = iqsynth.unit_vectors(2000, 128, 8, np.float64)
    for variant in (O.FULL, O.FAST, O.PLANAR2D):
        m = [O.mse(X, O.roundtrip(X, O.make_params(128, b, variant, 9))[0]) for b in (1, 2, 3, 4)]
        assert m[0] > m[1] > m[2] > m[3]


def test_codes_idempotent_whp():
    """Re-encoding x^ gives the same codes w.h.p. (x^ itself is rescaled by
    ||c||, so reconstruction is NOT idempotent — S:336 is false)."""
    X = iqsynth.unit_vectors(2000, 128, 10, np.float64)
    p = O.make_params(128, 3, O.FULL, 10)
    xh, codes, _, _ = O.roundtrip(X, p)
    codes2 = O.encode(xh, p)[0]
    assert np.mean(codes2 == codes) > 0.999


def test_outlier_channels_rotation_helps():
    """Rotation isotropizes unequal per-coordinate energy:
    MSE(Full) < MSE(identity); 4-D mixing beats 2-D."""
    X = iqsynth.outlier_vectors(6000, 128, 11, np.float64)
    for b in (2, 3):
        ident = O.mse(X, O.roundtrip(X, O.identity_params(128, b, O.FULL))[0])
        full = O.mse(X, O.roundtrip(X, O.make_params(128, b, O.FULL, 12))[0])
        fast = O.mse(X, O.roundtrip(X, O.make_params(128, b, O.FAST, 12))[0])
        planar = O.mse(X, O.roundtrip(X, O.make_params(128, b, O.PLANAR2D, 12))[0])
        assert full < ident and fast < ident
        assert full < planar and fast < planar
