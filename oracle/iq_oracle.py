"""IsoQuant stage-1 CPU ORACLE (fp64, NumPy) — TEST INFRASTRUCTURE ONLY.

This module is the plain, slow, obviously-correct statement of what the
IsoQuant stage-1 quantize -> dequantize path computes (arXiv 2603.28430,
Algorithm 1).  It exists to check the CUDA path, never to
serve it:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
  ``cpu_baseline`` leg and ``--impl reference`` arm) may import or execute it.
* It shares no code with ``paper_2603_28430_b200`` (the product) and imports
  nothing from it; the product imports nothing from here.  The only shared
  module is ``iqsynth`` (seeded synthetic inputs, no method arithmetic).
* Every step follows the paper in its order and notation.  Where the paper is
  silent the reading taken is the one listed in DESIGN.md "Readings" (R1..R18)
  and cited below as ``[Rn]``.

Citations: ``P:n`` = PAPER.md line n (LaTeX source of the paper); ``S:n`` =
SPEC.md line n (a CPU-program spec written from the paper; used only for
worked examples and interface ideas).

Parity pins: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (the paper's
printed numbers, the quaternion defining relations, closed forms, published
reference values, brute force).  Functions without such a pin say so in their
docstring ("parity unpinned"); there are none at present.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# Variants (Algorithm 1 REQUIRE line: mode in {Full, Fast, 2D})
# ----------------------------------------------------------------------------
FULL = 0      # IsoQuant-Full   T(v) = q_L v conj(q_R)
FAST = 1      # IsoQuant-Fast   T(v) = q_L v
PLANAR2D = 2  # 2-D special case u -> R(theta) u
VARIANT_NAMES = {FULL: "full", FAST: "fast", PLANAR2D: "planar2d"}

EPS = 1e-12   # epsilon of Alg. 1 line 1 "x / max(rho, eps)"; value [R5]

# ----------------------------------------------------------------------------
# Counter-based parameter RNG [R12]: SplitMix64 -> 53-bit uniforms ->
# Box-Muller.  The paper only says "sample the initial u vectors from a
# Gaussian distribution" and "Gaussian-normalize sampling on S^3 ...
# uniform angle sampling for the 2D special case"; the generator is
# ours.  Output k of SplitMix64 seeded with s is mix(s + (k+1)*GAMMA).
# ----------------------------------------------------------------------------
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_THETA_STREAM_KEY = 0x2D358DCCAA6C78A5   # angle stream: seed XOR this key [R12]
_RESAMPLE_STRIDE = 1 << 40               # counter offset per resample attempt


def splitmix64(seed: int, k: int) -> int:
    """k-th (0-based) output of SplitMix64 seeded with ``seed`` (Steele, Lea,
    Flood 2014; the standard constants).  Counter-based: no state is kept."""
    z = (seed + (k + 1) * _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniform01(seed: int, k: int) -> float:
    """Uniform in (0, 1]: ((out >> 11) + 1) * 2^-53  [R12]."""
    return ((splitmix64(seed, k) >> 11) + 1) * (1.0 / 9007199254740992.0)


def gaussian(seed: int, j: int) -> float:
    """j-th standard normal of the stream: Box-Muller on the uniform pair
    (2p, 2p+1), p = j // 2; even j takes the cosine branch, odd j the sine.
    Uses ``math`` (the C library), element by element."""
    p = j // 2
    u1 = uniform01(seed, 2 * p)
    u2 = uniform01(seed, 2 * p + 1)
    r = math.sqrt(-2.0 * math.log(u1))
    t = 2.0 * math.pi * u2
    return r * (math.cos(t) if (j % 2 == 0) else math.sin(t))


def _unit_quaternion(seed: int, j0: int) -> np.ndarray:
    """q = u / ||u||_2 with u ~ N(0, I_4) ("Gaussian-normalize
    sampling on S^3").  Gaussians j0..j0+3; resample (counter + 2^40) if
    ||u|| < 1e-12 (measure zero)."""
    attempt = 0
    while True:
        off = j0 + attempt * _RESAMPLE_STRIDE
        u = [gaussian(seed, off + c) for c in range(4)]
        nrm = math.sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2] + u[3] * u[3])
        if nrm >= 1e-12:
            return np.array([u[0] / nrm, u[1] / nrm, u[2] / nrm, u[3] / nrm])
        attempt += 1


def g4(d: int) -> int:
    """g = ceil(d / 4) quaternion blocks."""
    return -(-d // 4)


def g2(d: int) -> int:
    """g_2 = ceil(d / 2) planar blocks."""
    return -(-d // 2)


def make_rotation_params(d: int, variant: int, seed: int):
    """Random fixed block rotations [R12][R13].

    Full: (q_L^(i), q_R^(i)) for i < g, Gaussians 8i+0..3 (q_L) and 8i+4..7
    (q_R).  Fast: q_L^(i) only, from the same counters as Full's q_L, so
    Fast(seed) == Full(seed) with q_R := 1.  2D: theta_j = 2*pi*U_j from the
    angle stream, returned as (cos theta_j, sin theta_j) [R10].

    Returns (qL [g,4], qR [g,4] or None, cs [g2,2] or None), fp64.
    """
    if variant in (FULL, FAST):
        g = g4(d)
        qL = np.stack([_unit_quaternion(seed, 8 * i) for i in range(g)])
        qR = (np.stack([_unit_quaternion(seed, 8 * i + 4) for i in range(g)])
              if variant == FULL else None)
        return qL, qR, None
    if variant == PLANAR2D:
        s2 = seed ^ _THETA_STREAM_KEY
        cs = []
        for j in range(g2(d)):
            th = 2.0 * math.pi * uniform01(s2, j)
            cs.append((math.cos(th), math.sin(th)))
        return None, None, np.array(cs, dtype=np.float64).reshape(-1, 2)
    raise ValueError(f"unknown variant {variant}")


# ----------------------------------------------------------------------------
# Quaternion algebra: v = x0 + x1 i + x2 j + x3 k  [R8]
# ----------------------------------------------------------------------------
def qmul(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Hamilton product p*q over the last axis (components (a,b,c,d) =
    a + b i + c j + d k), from i^2 = j^2 = k^2 = ijk = -1.
    16 multiplications and 12 additions."""
    a1, b1, c1, d1 = p[..., 0], p[..., 1], p[..., 2], p[..., 3]
    a2, b2, c2, d2 = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([
        a1 * a2 - b1 * b2 - c1 * c2 - d1 * d2,
        a1 * b2 + b1 * a2 + c1 * d2 - d1 * c2,
        a1 * c2 - b1 * d2 + c1 * a2 + d1 * b2,
        a1 * d2 + b1 * c2 - c1 * b2 + d1 * a2,
    ], axis=-1)


def qconj(q: np.ndarray) -> np.ndarray:
    """conj(q) = a - b i - c j - d k."""
    return q * np.array([1.0, -1.0, -1.0, -1.0])


# ----------------------------------------------------------------------------
# Block transforms (Method; Algorithm 1 lines 3-13)
# ----------------------------------------------------------------------------
def forward_blocks(variant: int, qL, qR, cs, v: np.ndarray) -> np.ndarray:
    """Forward local rotation of every block.

    v: [..., g, 4] quaternion blocks (Full/Fast) or [..., g2, 2] pairs (2D).
    Full: v~ = q_L v conj(q_R) (Alg.1 l.5).
    Fast: v~ = q_L v          (Alg.1 l.9).
    2D:   u~ = R(theta) u      (Alg.1 l.13).
    """
    if variant == FULL:
        return qmul(qmul(qL, v), qconj(qR))
    if variant == FAST:
        return qmul(qL, v)
    if variant == PLANAR2D:
        c, s = cs[:, 0], cs[:, 1]
        u0, u1 = v[..., 0], v[..., 1]
        return np.stack([c * u0 - s * u1, s * u0 + c * u1], axis=-1)
    raise ValueError(variant)


def inverse_blocks(variant: int, qL, qR, cs, vh: np.ndarray) -> np.ndarray:
    """Inverse local rotation of every (quantized) block.

    Full: v_rec = conj(q_L) v^ q_R (Alg.1 l.7; inverse from the
          Proposition).
    Fast: v_rec = conj(q_L) v^     (Alg.1 l.11).
    2D:   u_rec = R(-theta) u^     (Alg.1 l.15).
    """
    if variant == FULL:
        return qmul(qmul(qconj(qL), vh), qR)
    if variant == FAST:
        return qmul(qconj(qL), vh)
    if variant == PLANAR2D:
        c, s = cs[:, 0], cs[:, 1]
        u0, u1 = vh[..., 0], vh[..., 1]
        return np.stack([c * u0 + s * u1, -s * u0 + c * u1], axis=-1)
    raise ValueError(variant)


def block_width(variant: int) -> int:
    """4-D blocks for Full/Fast, 2-D for the planar case (Alg.1 l.2)."""
    return 2 if variant == PLANAR2D else 4


# ----------------------------------------------------------------------------
# Scalar quantizer Q: Lloyd-Max for N(0,1), scaled by 1/sqrt(d) [R1][R2]
# ----------------------------------------------------------------------------
def _Phi(x: float) -> float:
    if x == math.inf:
        return 1.0
    if x == -math.inf:
        return 0.0
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


def _phi(x: float) -> float:
    if math.isinf(x):
        return 0.0
    return math.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)


def lloyd_max_gaussian(bits: int, tol: float = 1e-15, max_iter: int = 200000):
    """Lloyd-Max levels of a b-bit scalar quantizer for N(0,1) (P:16
    "per-coordinate Lloyd-Max quantization"; the fit is unspecified in the
    paper, [R1]).  Lloyd's iteration: thresholds = midpoints of adjacent
    levels, each level = conditional mean of its cell,
    c_k = (phi(t_k) - phi(t_{k+1})) / (Phi(t_{k+1}) - Phi(t_k)).
    Start: levels at the quantiles Phi^-1((k + 1/2) / L).  Stop when the
    largest level move is < tol.  Finally symmetrize exactly [R2]:
    c_{L-1-k} = -c_k.  Returns (levels fp64 [L], distortion D = E(z-Q(z))^2).
    """
    from scipy.special import ndtri  # quantile only seeds the iteration
    L = 1 << bits
    c = [float(ndtri((k + 0.5) / L)) for k in range(L)]
    for _ in range(max_iter):
        t = [-math.inf] + [0.5 * (c[k] + c[k + 1]) for k in range(L - 1)] + [math.inf]
        new = []
        for k in range(L):
            a, b = t[k], t[k + 1]
            new.append((_phi(a) - _phi(b)) / (_Phi(b) - _Phi(a)))
        delta = max(abs(new[k] - c[k]) for k in range(L))
        c = new
        if delta < tol:
            break
    h = L // 2
    pos = [0.5 * (c[h + m] - c[h - 1 - m]) for m in range(h)]
    c = [-pos[h - 1 - k] for k in range(h)] + pos
    # distortion E[(z - Q(z))^2] = 1 - sum_k c_k^2 P_k  (centroid condition)
    t = [-math.inf] + [0.5 * (c[k] + c[k + 1]) for k in range(L - 1)] + [math.inf]
    dist = 1.0 - sum(c[k] * c[k] * (_Phi(t[k + 1]) - _Phi(t[k])) for k in range(L))
    return np.array(c), dist


@dataclass
class Codebook:
    """The shared scalar codebook of one (d, b) configuration [R1][R2].

    ``centroids`` are fp32 values (stored in fp64): round_fp32(c_k / sqrt(d))
    — the codebook as a device stores it [R14b].
    ``thresholds`` are the fp64 midpoints (C_k + C_{k+1}) / 2 of adjacent
    centroids (exact in fp64: both are fp32 values) — the decision boundaries
    of nearest-centroid assignment, NOT rounded to fp32: the oracle
    decides in fp64 [R14b].
    """
    bits: int
    d: int
    centroids: np.ndarray    # [L] fp32-representable, dtype float64
    thresholds: np.ndarray   # [L-1] dtype float64, exact midpoints
    levels_unit: np.ndarray  # [L] fp64 N(0,1) Lloyd-Max levels


def make_codebook(d: int, bits: int) -> Codebook:
    """Lloyd-Max N(0,1) levels scaled by 1/sqrt(d) (a unit vector's rotated
    coordinates have variance 1/d, P:269-273 with k=d) [R1]."""
    levels, _ = lloyd_max_gaussian(bits)
    C32 = (levels / math.sqrt(d)).astype(np.float32)
    C = C32.astype(np.float64)
    T = (C[:-1] + C[1:]) * 0.5
    return Codebook(bits=bits, d=d, centroids=C, thresholds=T, levels_unit=levels)


def quantize_codes(y: np.ndarray, cb: Codebook) -> np.ndarray:
    """Nearest-centroid code of every coordinate (v^ = Q(v~); Alg.1
    l.6), written as the count over the sorted thresholds t_k (the
    midpoints of adjacent centroids):

        code = #{k : y >= t_k}

    in fp64 on the fp64 rotated coordinate [R14b].  This is argmin_k
    |y - C_k| except at an exact midpoint, where the paper is silent
    (P:182); reading [R3] takes the upper code there, so y = +-0
    codes on the positive side (-0 >= 0).  Values beyond the extreme
    thresholds clamp to the end codes [R4] (automatic with counting)."""
    y = np.asarray(y, dtype=np.float64)
    codes = np.zeros(y.shape, dtype=np.int64)
    for t in cb.thresholds:
        codes += (y >= t)
    return codes


def dequantize_codes(codes: np.ndarray, cb: Codebook) -> np.ndarray:
    """v^ = C[code] (decoder lookup)."""
    return cb.centroids[codes]


# ----------------------------------------------------------------------------
# Bit packing [R7] (not in the paper)
# ----------------------------------------------------------------------------
def pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """LSB-first bitstream per row: bit (j*b + m) of the row stream is bit m
    of code_j; byte B holds stream bits 8B .. 8B+7 (bit 8B in its LSB).
    codes: [n, m] ints < 2^b -> [n, ceil(m*b/8)] uint8.  Bit by bit."""
    codes = np.asarray(codes, dtype=np.int64)
    n, m = codes.shape
    nbytes = -(-m * bits // 8)
    out = np.zeros((n, nbytes), dtype=np.uint8)
    for j in range(m):
        for k in range(bits):
            pos = j * bits + k
            bit = ((codes[:, j] >> k) & 1).astype(np.uint8)
            out[:, pos // 8] |= (bit << (pos % 8)).astype(np.uint8)
    return out


def unpack_codes(packed: np.ndarray, bits: int, m: int) -> np.ndarray:
    """Inverse of ``pack_codes``: [n, nbytes] uint8 -> [n, m] int64."""
    packed = np.asarray(packed, dtype=np.uint8)
    n = packed.shape[0]
    codes = np.zeros((n, m), dtype=np.int64)
    for j in range(m):
        for k in range(bits):
            pos = j * bits + k
            bit = (packed[:, pos // 8] >> (pos % 8)) & 1
            codes[:, j] |= bit.astype(np.int64) << k
    return codes


def code_bytes_per_vector(d: int, bits: int, variant: int = FULL) -> int:
    """Packed code bytes per row: ceil(padded_len * b / 8) [R7]."""
    bw = block_width(variant)
    padded = -(-d // bw) * bw
    return -(-padded * bits // 8)


# ----------------------------------------------------------------------------
# Parameters of one configuration
# ----------------------------------------------------------------------------
@dataclass
class OracleParams:
    d: int
    bits: int
    variant: int
    seed: int
    qL: np.ndarray = None
    qR: np.ndarray = None
    cs: np.ndarray = None
    cb: Codebook = None

    @property
    def L(self) -> int:
        return 1 << self.bits


def make_params(d: int, bits: int, variant: int, seed: int) -> OracleParams:
    """Random fixed rotations + the shared codebook [R1]."""
    qL, qR, cs = make_rotation_params(d, variant, seed)
    return OracleParams(d=d, bits=bits, variant=variant, seed=seed,
                        qL=qL, qR=qR, cs=cs, cb=make_codebook(d, bits))


def identity_params(d: int, bits: int, variant: int) -> OracleParams:
    """q_L = q_R = 1 and theta = 0: every transform is the identity."""
    p = OracleParams(d=d, bits=bits, variant=variant, seed=-1, cb=make_codebook(d, bits))
    one = np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (g4(d), 1))
    if variant in (FULL, FAST):
        p.qL = one.copy()
        p.qR = one.copy() if variant == FULL else None
    else:
        p.cs = np.tile(np.array([1.0, 0.0]), (g2(d), 1))
    return p


# ----------------------------------------------------------------------------
# Algorithm 1
# ----------------------------------------------------------------------------
def _as_f64(X) -> np.ndarray:
    X = np.asarray(X)
    if X.ndim != 2:
        raise ValueError("X must be [n, d]")
    return X.astype(np.float64)


def _partition(xbar: np.ndarray, p: OracleParams) -> np.ndarray:
    """Alg.1 l.2: zero-pad to g*w and view as [n, g, w] blocks;
    consecutive coordinates form a block [R8][R9]; zero padding."""
    n, d = xbar.shape
    w = block_width(p.variant)
    g = -(-d // w)
    padded = np.zeros((n, g * w))
    padded[:, :d] = xbar
    return padded.reshape(n, g, w)


def encode(X, p: OracleParams):
    """Encoder half of Algorithm 1: returns (codes [n, padded] int64,
    packed [n, bytes] uint8, rho [n] fp64).

    l.1  rho = ||x||_2, xbar = x / max(rho, eps)
    l.2  partition into zero-padded blocks
    l.3-13  per block: forward rotation, then Q
    """
    X = _as_f64(X)
    rho = np.sqrt(np.sum(X * X, axis=1))                       # l.1
    xbar = X / np.maximum(rho, EPS)[:, None]                    # l.1
    blocks = _partition(xbar, p)                                # l.2
    vt = forward_blocks(p.variant, p.qL, p.qR, p.cs, blocks)    # l.5/9/13
    y = vt.reshape(X.shape[0], -1)
    codes = quantize_codes(y, p.cb)                             # l.6/10/14
    packed = pack_codes(codes, p.bits)
    return codes, packed, rho


def decode(codes: np.ndarray, rho: np.ndarray, p: OracleParams) -> np.ndarray:
    """Decoder half of Algorithm 1: v^ = C[code], inverse block
    rotation, concatenate, drop padding (l.17), x^ = rho * (...)
    (l.18; the stored rho itself is used, [R5])."""
    n = codes.shape[0]
    w = block_width(p.variant)
    vh = dequantize_codes(codes, p.cb).reshape(n, -1, w)
    vrec = inverse_blocks(p.variant, p.qL, p.qR, p.cs, vh)      # l.7/11/15
    xr = vrec.reshape(n, -1)[:, :p.d]                            # l.17
    return np.asarray(rho, dtype=np.float64)[:, None] * xr      # l.18


def decode_packed(packed: np.ndarray, rho: np.ndarray, p: OracleParams) -> np.ndarray:
    """Decode from the packed byte format (unpack, then ``decode``)."""
    w = block_width(p.variant)
    m = -(-p.d // w) * w
    return decode(unpack_codes(packed, p.bits, m), rho, p)


def roundtrip(X, p: OracleParams):
    """x^ = D(Q(E(x))) via Algorithm 1.  Returns
    (x_hat fp64 [n,d], codes [n,padded], packed uint8, rho fp64)."""
    codes, packed, rho = encode(X, p)
    return decode(codes, rho, p), codes, packed, rho


def rotated_coordinates(X, p: OracleParams) -> np.ndarray:
    """y = T(xbar) in fp64 (before Q) — used by parity tests to locate
    decision boundaries (distance of y to the nearest threshold)."""
    X = _as_f64(X)
    rho = np.sqrt(np.sum(X * X, axis=1))
    xbar = X / np.maximum(rho, EPS)[:, None]
    vt = forward_blocks(p.variant, p.qL, p.qR, p.cs, _partition(xbar, p))
    return vt.reshape(X.shape[0], -1)


def mse(X, X_hat) -> float:
    """Reconstruction MSE: mean over n*d of (x - x^)^2 [R17]."""
    X = _as_f64(X)
    return float(np.mean((X - np.asarray(X_hat, dtype=np.float64)) ** 2))


# ----------------------------------------------------------------------------
# Complexity model (Section "Complexity Analysis", Table 1)
# ----------------------------------------------------------------------------
class _CountingScalar:
    """A scalar that counts multiplications performed on it: used to *count*
    the FMAs of the oracle's own transform instead of restating a formula."""
    muls = 0

    def __init__(self, v=0.0):
        self.v = v

    def __mul__(self, o):
        _CountingScalar.muls += 1
        return _CountingScalar(self.v * (o.v if isinstance(o, _CountingScalar) else o))

    __rmul__ = __mul__

    def _lin(self, o, f):
        return _CountingScalar(f(self.v, o.v if isinstance(o, _CountingScalar) else o))

    def __add__(self, o):
        return self._lin(o, lambda a, b: a + b)

    __radd__ = __add__

    def __sub__(self, o):
        return self._lin(o, lambda a, b: a - b)

    def __rsub__(self, o):
        return self._lin(o, lambda a, b: b - a)

    def __neg__(self):
        return _CountingScalar(-self.v)


def complexity(variant: int, d: int):
    """(params, forward-rotation FMAs) of one vector, counted by running the
    oracle's own forward transform on counting scalars, with the paper's
    convention "16 mult + 12 add ~ 16 FMA": one FMA per scalar
    multiplication of a parameter by a coordinate-dependent value.
    Params = stored scalars: Full 8 per block, Fast 4, 2D 2 (cos, sin) [R10].
    Compared against Table 1 and P:333 in tests."""
    p = make_params(d, 1, variant, seed=0) if variant != PLANAR2D else None
    if variant == PLANAR2D:
        qL, qR, cs = make_rotation_params(d, variant, 0)
        nparams = cs.size
        blocks = g2(d)
        obj = np.empty((1, 2), dtype=object)
        obj[0, 0], obj[0, 1] = _CountingScalar(0.3), _CountingScalar(0.7)
        csobj = np.empty((1, 2), dtype=object)
        csobj[0, 0], csobj[0, 1] = cs[0, 0], cs[0, 1]
        _CountingScalar.muls = 0
        forward_blocks(PLANAR2D, None, None, csobj, obj[None, :, :].reshape(1, 1, 2))
        return nparams, _CountingScalar.muls * blocks
    qL, qR = p.qL, p.qR
    nparams = qL.size + (qR.size if qR is not None else 0)
    blocks = g4(d)
    v = np.empty((1, 1, 4), dtype=object)
    for c in range(4):
        v[0, 0, c] = _CountingScalar(0.1 * (c + 1))
    _CountingScalar.muls = 0
    forward_blocks(variant, qL[:1], None if qR is None else qR[:1], None, v)
    return nparams, _CountingScalar.muls * blocks


# ----------------------------------------------------------------------------
# Closed-form expectation used as a pin (P:277-279 with k = d)
# ----------------------------------------------------------------------------
def sphere_marginal_pdf(k: int, z):
    """Marginal density of one coordinate of a uniform point on S^{k-1}:
    f_k(z) = Gamma(k/2) / (sqrt(pi) Gamma((k-1)/2)) (1 - z^2)^((k-3)/2)
    (normalisation is the Beta(1/2,(k-1)/2) constant)."""
    z = np.asarray(z, dtype=np.float64)
    logc = math.lgamma(k / 2.0) - 0.5 * math.log(math.pi) - math.lgamma((k - 1) / 2.0)
    return np.exp(logc) * np.power(np.clip(1.0 - z * z, 0.0, None), (k - 3) / 2.0)


def expected_unit_vector_mse(d: int, bits: int) -> float:
    """E[(z - Q(z))^2] for z ~ f_d with this build's fp32 codebook: the
    per-coordinate MSE of stage 1 on unit vectors uniform on S^{d-1}, for ANY
    fixed orthogonal block rotation (the rotated vector is again uniform on
    the sphere, so every coordinate has marginal f_d).  Computed
    by adaptive quadrature cell by cell."""
    from scipy.integrate import quad
    cb = make_codebook(d, bits)
    C = cb.centroids
    T = cb.thresholds.astype(np.float64)
    edges = [-1.0] + list(T) + [1.0]
    total = 0.0
    for k in range(len(C)):
        a, b = edges[k], edges[k + 1]
        val, _ = quad(lambda z: (z - C[k]) ** 2 * float(sphere_marginal_pdf(d, z)),
                      a, b, epsabs=1e-15, epsrel=1e-12, limit=200)
        total += val
    return total
