"""GPU-vs-oracle parity checks with the north-star tolerances (BASELINE.json):
codes agree on >= 99.99% of coordinates and every mismatch lies within 1e-5
of a decision threshold; norms within 1e-6 relative; reconstructions within
1e-5 (fp32) / 2e-3 (fp16) relative per vector; MSE within 0.5% of the
oracle's.  Test infrastructure (imports the oracle)."""
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


def assert_parity(r: ParityReport, dtype, check_mse: bool = True):
    tol = RECON_RTOL[dtype]
    assert r.code_agreement >= CODE_AGREEMENT, r
    assert r.max_boundary_dist <= BOUNDARY, r
    assert r.max_norm_rel <= NORM_RTOL, r
    assert r.max_recon_rel <= tol, r
    assert r.max_recon_rel_all <= tol, r
    if check_mse and r.mse_oracle > 0:
        assert abs(r.mse_gpu - r.mse_oracle) <= MSE_RTOL * r.mse_oracle, r
