"""Learning the block rotations, CPU ORACLE (fp64, NumPy) — TEST
INFRASTRUCTURE ONLY (same rules as ``iq_oracle``).

PAPER.md "Parameterization and Learning": each unit quaternion
is q = u / ||u|| with a free u in R^4, "keeping optimization in Euclidean
space".  The paper names no objective; reading R29 takes the
stage-1 distortion on normalised rows,

    L = sum_rows sum_j ( ybar_j - Q(ybar_j) )^2,   ybar = T(x / max(rho, eps)),

(the normalised reconstruction error, since T is orthogonal).  Q is
piecewise constant, so L is differentiable almost everywhere with

    dL/d ybar = 2 e,  e = ybar - Q(ybar).

This module states that gradient twice, independently:
* ``operator_grad``: dL/dM_b = 2 sum_rows e_b xbar_b^T for the block operator
  M_b (ybar_b = M_b xbar_b), the quantity the GPU kernel accumulates;
* ``rot_grad``: dL/dq by the chain rule through the Hamilton products of the
  paper's map (Full q_L v conj(q_R), Fast q_L v, 2D R(theta)), projected on
  the tangent space of each unit vector (R30: the gradient with respect to u
  at ||u|| = 1).
Pins (tests/test_oracle_learn.py): central finite differences of L in u and
in M, Fast = Full with q_R = 1, agreement of the two statements, a descent
step lowering L.
"""
from __future__ import annotations

import numpy as np

from . import iq_oracle as O


def _blocks(X, p: O.OracleParams):
    """xbar and ybar as [n, g, w] blocks (Alg.1 l.1-2) and the quantization
    error e = ybar - Q(ybar) in the same layout (decisions as in iq_oracle)."""
    X = np.asarray(X).astype(np.float64)
    rho = np.sqrt(np.sum(X * X, axis=1))
    xbar = X / np.maximum(rho, O.EPS)[:, None]
    xb = O._partition(xbar, p)
    yb = O.forward_blocks(p.variant, p.qL, p.qR, p.cs, xb)
    n = X.shape[0]
    y = yb.reshape(n, -1)
    c = O.dequantize_codes(O.quantize_codes(y, p.cb), p.cb)
    e = (y - c).reshape(yb.shape)
    return xb, yb, e


def distortion(X, p: O.OracleParams) -> float:
    """L = sum over rows and coordinates of (ybar - Q(ybar))^2 (R29)."""
    _, _, e = _blocks(X, p)
    return float(np.sum(e * e))


def operator_grad(X, p: O.OracleParams) -> np.ndarray:
    """dL/dM_b = 2 sum_rows e_b xbar_b^T, [g, w, w] (row index = output)."""
    xb, _, e = _blocks(X, p)
    return 2.0 * np.einsum("ngi,ngj->gij", e, xb)


def _project(gq: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Tangent projection g - (g.q) q per unit vector (rows of q)."""
    return gq - np.sum(gq * q, axis=-1, keepdims=True) * q


def rot_grad(X, p: O.OracleParams) -> np.ndarray:
    """dL/d(rotation parameters) in the iq_export_params layout, by the chain
    rule through the Hamilton products (R30).  Full: [g, 8] = (dq_L, dq_R);
    Fast: [g, 4]; 2D: [g2, 2] = (dc, ds), each projected on its tangent."""
    xb, _, e = _blocks(X, p)
    if p.variant == O.PLANAR2D:
        u0, u1 = xb[..., 0], xb[..., 1]
        gc = 2.0 * np.sum(e[..., 0] * u0 + e[..., 1] * u1, axis=0)     # d/dc of (c u0 - s u1, s u0 + c u1)
        gs = 2.0 * np.sum(-e[..., 0] * u1 + e[..., 1] * u0, axis=0)
        return _project(np.stack([gc, gs], axis=-1), p.cs).reshape(-1)
    g = xb.shape[1]
    E = np.eye(4)
    gl = np.zeros((g, 4))
    gr = np.zeros((g, 4))
    for k in range(4):
        ek = np.tile(E[k], (g, 1))
        if p.variant == O.FULL:
            dyl = O.qmul(O.qmul(ek, xb), O.qconj(p.qR))               # d ybar / d q_L[k]
            dyr = O.qmul(O.qmul(p.qL, xb), O.qconj(ek))               # d ybar / d q_R[k]
            gr[:, k] = 2.0 * np.sum(e * dyr, axis=(0, 2))
        else:
            dyl = O.qmul(ek, xb)
        gl[:, k] = 2.0 * np.sum(e * dyl, axis=(0, 2))
    gl = _project(gl, p.qL)
    if p.variant == O.FULL:
        return np.concatenate([gl, _project(gr, p.qR)], axis=1).reshape(-1)
    return gl.reshape(-1)


def params_from_rot(d: int, bits: int, variant: int, rot) -> O.OracleParams:
    """OracleParams from explicit parameters in the export layout, each unit
    vector normalised (q = u / ||u||)."""
    rot = np.asarray(rot, dtype=np.float64)
    p = O.OracleParams(d=d, bits=bits, variant=variant, seed=-1, cb=O.make_codebook(d, bits))
    if variant == O.PLANAR2D:
        cs = rot.reshape(-1, 2)
        p.cs = cs / np.linalg.norm(cs, axis=1, keepdims=True)
    elif variant == O.FULL:
        r = rot.reshape(-1, 8)
        p.qL = r[:, :4] / np.linalg.norm(r[:, :4], axis=1, keepdims=True)
        p.qR = r[:, 4:] / np.linalg.norm(r[:, 4:], axis=1, keepdims=True)
    else:
        r = rot.reshape(-1, 4)
        p.qL = r / np.linalg.norm(r, axis=1, keepdims=True)
    return p


def rot_of(p: O.OracleParams) -> np.ndarray:
    """The export-layout parameter vector of p."""
    if p.variant == O.PLANAR2D:
        return p.cs.reshape(-1).copy()
    if p.variant == O.FULL:
        return np.concatenate([p.qL, p.qR], axis=1).reshape(-1)
    return p.qL.reshape(-1).copy()
