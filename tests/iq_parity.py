"""GPU-vs-oracle parity checks with the north-star tolerances (BASELINE.json):
codes agree on >= 99.99% of coordinates and every mismatch lies within 1e-5
of a decision threshold; norms within 1e-6 relative; reconstructions within
1e-5 (fp32) / 2e-3 (fp16) relative per vector; MSE within 0.5% of the
oracle's.  Test infrastructure (imports the oracle).

Three entry points, one per kind of kernel output:

* ``check``        -- a reconstruction WITH the codes and norms the kernel
                      emitted (quantize K1, fused + codes K3'),
* ``check_values`` -- a reconstruction ALONE (the fused kernel as benchmarked,
                      K3 without code emission): the codes it was built from
                      are recovered by the oracle's own forward rotation of
                      x^ / rho and a nearest-centroid search, then held to the
                      same code / boundary / per-row bars as ``check``,
* ``check_decode`` -- the dequantizer K2 on given codes and norms: no decision
                      is involved, so every row must match the oracle's decode
                      of those codes.

No row is exempt from any bar."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle import iq_oracle as O

CODE_AGREEMENT = 0.9999
BOUNDARY = 1e-5
NORM_RTOL = 1e-6
# bf16 (R28): the fp16 bound scaled by the 4x coarser output rounding
RECON_RTOL = {np.float32: 1e-5, np.float16: 2e-3, "bf16": 8e-3}
MSE_RTOL = 5e-3


@dataclass
class ParityReport:
    n: int
    code_agreement: float
    n_code_mismatch: int
    max_boundary_dist: float
    max_norm_rel: float
    max_recon_rel: float
    max_recon_rel_all: float
    mse_gpu: float
    mse_oracle: float


def _rel_rows(a, b):
    num = np.linalg.norm(a - b, axis=1)
    den = np.linalg.norm(b, axis=1)
    out = np.zeros_like(num)
    nz = den > 0
    out[nz] = num[nz] / den[nz]
    out[~nz] = num[~nz]
    return out


def check(X: np.ndarray, po: O.OracleParams, y_gpu: np.ndarray, codes_gpu: np.ndarray,
          norms_gpu: np.ndarray, dtype, strict_rows=None) -> ParityReport:
    """Compare GPU outputs for input rows X (as stored) with the oracle.
    ``strict_rows``: boolean mask of rows the reconstruction bound applies to
    (default: rows with rho >= 1e-12, [R5])."""
    n, d = X.shape
    xh_o, codes_o, _, rho_o = O.roundtrip(X, po)
    m = codes_o.shape[1]
    codes_g = O.unpack_codes(codes_gpu, po.bits, m)
    mism = codes_g != codes_o
    agree = 1.0 - mism.mean() if mism.size else 1.0
    maxdist = 0.0
    if mism.any():
        y = O.rotated_coordinates(X, po)[mism]
        T = po.cb.thresholds.astype(np.float64)
        maxdist = float(np.max(np.min(np.abs(y[:, None] - T[None, :]), axis=1)))
    norm_rel = np.abs(norms_gpu.astype(np.float64) - rho_o) / np.maximum(rho_o, 1e-30)
    norm_rel[rho_o == 0] = np.abs(norms_gpu[rho_o == 0])
    y64 = y_gpu.astype(np.float64)
    rel = _rel_rows(y64, xh_o)
    if strict_rows is None:
        strict_rows = rho_o >= 1e-12
    clean = strict_rows & ~mism.any(axis=1)
    # every row: oracle decode of the GPU's own codes and norms
    xh_from_gpu = O.decode(codes_g, norms_gpu.astype(np.float64), po)
    rel_all = _rel_rows(y64, xh_from_gpu)
    mse_g = float(np.mean((X.astype(np.float64) - y64) ** 2))
    mse_o = float(np.mean((X.astype(np.float64) - xh_o) ** 2))
    return ParityReport(
        n=n, code_agreement=float(agree), n_code_mismatch=int(mism.sum()),
        max_boundary_dist=maxdist,
        max_norm_rel=float(norm_rel[strict_rows].max()) if strict_rows.any() else 0.0,
        max_recon_rel=float(rel[clean].max()) if clean.any() else 0.0,
        max_recon_rel_all=float(rel_all[strict_rows].max()) if strict_rows.any() else 0.0,
        mse_gpu=mse_g, mse_oracle=mse_o)


def _rotate_rows(Y: np.ndarray, po: O.OracleParams) -> np.ndarray:
    """T(y) per row with the oracle's block rotation (no normalisation)."""
    n = Y.shape[0]
    return O.forward_blocks(po.variant, po.qL, po.qR, po.cs, O._partition(Y, po)).reshape(n, -1)


def implied_codes(y64: np.ndarray, rho: np.ndarray, po: O.OracleParams):
    """The codes a reconstruction x^ = rho * T^-1(C[code]) was built from:
    z = T(x^ / rho) (T orthogonal) and the nearest centroid.
    Returns (codes, max |z - C[code]| / half the smallest centroid gap): the
    second number is ~1e-3 for an fp16 reconstruction and must stay well below
    1, else the output is not a reconstruction from any codes."""
    C = po.cb.centroids
    z = _rotate_rows(y64 / np.maximum(rho, 1e-300)[:, None], po)
    k = np.argmin(np.abs(z[..., None] - C), axis=-1)
    half_gap = 0.5 * float(np.min(np.diff(C))) if len(C) > 1 else 1.0
    resid = float(np.max(np.abs(z - C[k]))) / half_gap if z.size else 0.0
    return k, resid


def check_values(X: np.ndarray, po: O.OracleParams, y_gpu: np.ndarray, dtype):
    """Parity of a value-only reconstruction (no codes emitted) with the
    oracle.  Rows with rho >= 1e-12 [R5] are checked through their implied
    codes (code agreement, boundary distance of every mismatch, per-row error
    against the oracle's x^ where the codes agree and against the oracle's
    decode of the implied codes everywhere); zero rows must be exactly zero.
    Returns (ParityReport with the oracle's norms in place of the kernel's,
    max implied-code residual, zero rows all exact)."""
    n, d = X.shape
    _, codes_o, _, rho_o = O.roundtrip(X, po)
    y64 = y_gpu.astype(np.float64)
    strict = rho_o >= 1e-12
    codes_g = codes_o.copy()
    resid = 0.0
    if strict.any():
        codes_g[strict], resid = implied_codes(y64[strict], rho_o[strict], po)
    zero_ok = bool(np.all(y64[rho_o == 0] == 0.0))
    packed_g = O.pack_codes(codes_g, po.bits)
    r = check(X, po, y_gpu, packed_g, rho_o.astype(np.float32), dtype, strict_rows=strict)
    r.max_norm_rel = 0.0          # value-only output: no norms emitted
    return r, resid, zero_ok


def assert_values(res, dtype, check_mse: bool = True):
    r, resid, zero_ok = res
    assert zero_ok, "zero rows must reconstruct to exact zeros (S:312)"
    assert resid <= 0.25, f"output is not a reconstruction from any codes: residual {resid}"
    assert_parity(r, dtype, check_mse=check_mse)


def check_decode(codes_gpu: np.ndarray, norms_gpu: np.ndarray, y_gpu: np.ndarray, po: O.OracleParams):
    """Per-row relative error of the dequantizer's output against the
    oracle's decode (Alg.1 l.15-18) of the same codes and norms."""
    w = O.block_width(po.variant)
    m = -(-po.d // w) * w
    want = O.decode(O.unpack_codes(codes_gpu, po.bits, m), norms_gpu.astype(np.float64), po)
    rel = _rel_rows(y_gpu.astype(np.float64), want)
    return float(rel.max()) if rel.size else 0.0


def assert_parity(r: ParityReport, dtype, check_mse: bool = True):
    tol = RECON_RTOL[dtype]
    assert r.code_agreement >= CODE_AGREEMENT, r
    assert r.max_boundary_dist <= BOUNDARY, r
    assert r.max_norm_rel <= NORM_RTOL, r
    assert r.max_recon_rel <= tol, r
    assert r.max_recon_rel_all <= tol, r
    if check_mse and r.mse_oracle > 0:
        assert abs(r.mse_gpu - r.mse_oracle) <= MSE_RTOL * r.mse_oracle, r
