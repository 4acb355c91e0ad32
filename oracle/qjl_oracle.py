"""IsoQuant stage-2 residual sketch, CPU ORACLE (fp64, NumPy) — TEST
INFRASTRUCTURE ONLY (same rules as ``iq_oracle``: only tests/, smoke() and
bench.py's CPU legs may use it; it shares no code with the product).

The paper fixes only the residual and the kind of correction (section
"Compatibility with Residual Correction"):

    r = x - x^_mse,  projected with a quantized Johnson-Lindenstrauss
    transform (QJL) "or a related low-bit correction mechanism".

Everything below the residual is the QJL construction as DESIGN.md reads it
(R20-R24):

* R20  S in R^{m x d}, m = d, i.i.d. N(0, 1) from the parameter generator
       [R12] keyed with seed ^ QJL_STREAM_KEY, S[i][k] = N_(i*d + k), each
       rounded to IEEE half (round to nearest even).  The rounded values ARE
       the sketch.
* R21  r = x - x^, x^ the stage-1 reconstruction of ``iq_oracle``.
* R22  q_i = +1 if (S r)_i >= 0 else -1 (z = 0 -> +1).
* R23  gamma = ||r||_2.
* R24  <y, x> ~= <y, x^> + sqrt(pi/2)/m * gamma * <S y, q>, and
       x~ = x^ + sqrt(pi/2)/m * gamma * S^T q  (unbiased over S).

Parity pins (tests/test_oracle_qjl.py): the standard-normal law of S; the
sign of a one-hot residual is the sign of S's column (brute force); bits by
explicit loops on tiny inputs; unbiasedness of the estimator and of x~ by
Monte Carlo over sketch seeds against the closed forms E[<s,y> sign<s,r>] =
sqrt(2/pi) <y,r>/||r||; the variance bound of QJL; zero residual.
"""
from __future__ import annotations

import math

import numpy as np

from . import iq_oracle as O

QJL_STREAM_KEY = 0x514A4C534B455443   # R20


def sketch_matrix(d: int, seed: int, m: int | None = None) -> np.ndarray:
    """S [m, d] fp64 holding fp16-rounded standard normals (R20).  Element
    (i, k) is Gaussian number i*d + k of the keyed stream, element by
    element with ``iq_oracle.gaussian``."""
    m = d if m is None else m
    s = (seed ^ QJL_STREAM_KEY) & ((1 << 64) - 1)
    g = np.array([O.gaussian(s, j) for j in range(m * d)], dtype=np.float64)
    return g.astype(np.float16).astype(np.float64).reshape(m, d)


def sketch_bits(R: np.ndarray, S: np.ndarray) -> np.ndarray:
    """q in {0, 1}^[n, m], 1 meaning +1: [ (S r)_i >= 0 ] (R22)."""
    Z = np.asarray(R, dtype=np.float64) @ S.T
    return (Z >= 0).astype(np.uint8)


def pack_bits(q01: np.ndarray) -> np.ndarray:
    """LSB-first per row (bit i of the row stream = q_i), as the stage-1
    codes with one bit per symbol."""
    return O.pack_codes(q01.astype(np.int64), 1)


def unpack_bits(packed: np.ndarray, m: int) -> np.ndarray:
    return O.unpack_codes(packed, 1, m).astype(np.uint8)


def encode(X, p: O.OracleParams, S: np.ndarray):
    """Stage 1 + stage 2: returns (codes, packed, rho, x_hat, q01, gamma).
    r = x - x^ (R21, fp64), gamma = ||r|| (R23), q = [S r >= 0] (R22)."""
    X = np.asarray(X).astype(np.float64)
    x_hat, codes, packed, rho = O.roundtrip(X, p)
    R = X - x_hat
    gamma = np.sqrt(np.sum(R * R, axis=1))
    return codes, packed, rho, x_hat, sketch_bits(R, S), gamma


def correction(q01: np.ndarray, gamma: np.ndarray, S: np.ndarray) -> np.ndarray:
    """sqrt(pi/2)/m * gamma * S^T q (R24): the stage-2 estimate of r."""
    m = S.shape[0]
    q = 2.0 * np.asarray(q01, dtype=np.float64) - 1.0
    return (math.sqrt(math.pi / 2.0) / m) * np.asarray(gamma, dtype=np.float64)[:, None] * (q @ S)


def inner_product(Y, x_hat, q01, gamma, S) -> np.ndarray:
    """Row-wise estimate of <y_i, x_i> (R24):
    <y, x^> + sqrt(pi/2)/m * gamma * <S y, q>."""
    Y = np.asarray(Y, dtype=np.float64)
    m = S.shape[0]
    q = 2.0 * np.asarray(q01, dtype=np.float64) - 1.0
    sy = Y @ S.T
    return (np.sum(Y * x_hat, axis=1)
            + (math.sqrt(math.pi / 2.0) / m) * np.asarray(gamma) * np.sum(sy * q, axis=1))
