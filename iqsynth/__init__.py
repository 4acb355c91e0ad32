"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NO arithmetic of the IsoQuant method: it only
draws input vectors with the shape and distribution of the paper's workload
("synthetic normalized vectors") and a secondary test-only
distribution.  Recipe:

* isotropic: g ~ N(0, I_d) (NumPy PCG64, or torch's CUDA generator for the
  large device-resident configs), x = g / ||g||_2 computed in fp64 (host) or
  fp32 (device), THEN cast to the storage dtype (fp16 or fp32).  fp16 rows
  therefore have norm 1 +- ~1e-4, which exercises the norm split.
* outlier channels (tests only): rows g * s with s_j = 4 for j = 0 mod 4 and
  1 otherwise, then normalised — unequal per-coordinate energy, the case the
  paper's decorrelation argument is about.
* seeds: a global batch is cut into chunks of 2^16 rows; chunk c of the batch
  with base seed s is drawn from its own seed chunk_seed(s, c) (a SeedSequence
  hash of the pair, so no two (s, c) share a stream), and any rank can
  regenerate any chunk: the global batch is identical at every GPU count
  (``device_unit_vectors(..., row0=...)`` draws global rows [row0, row0+n)).
"""
from __future__ import annotations

import numpy as np

PARAMS_SEED = 20260331          # parameter seed used by bench and tests
CHUNK_ROWS = 1 << 16


def data_seed(config: int, chunk: int = 0) -> int:
    return 1000 * config + chunk


def unit_vectors(n: int, d: int, seed: int, dtype=np.float32) -> np.ndarray:
    """[n, d] rows uniform on S^{d-1} (normalised in fp64, then cast)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    g = rng.standard_normal((n, d))
    nrm = np.sqrt(np.sum(g * g, axis=1, keepdims=True))
    nrm[nrm == 0] = 1.0
    return (g / nrm).astype(dtype)


def outlier_vectors(n: int, d: int, seed: int, dtype=np.float32, scale: float = 4.0) -> np.ndarray:
    """[n, d] rows with one high-energy channel per 4-block, normalised."""
    rng = np.random.Generator(np.random.PCG64(seed))
    g = rng.standard_normal((n, d))
    s = np.ones(d)
    s[0::4] = scale
    g = g * s
    nrm = np.sqrt(np.sum(g * g, axis=1, keepdims=True))
    return (g / nrm).astype(dtype)


def gaussian_rows(n: int, d: int, seed: int, dtype=np.float32, sigma: float = 1.0) -> np.ndarray:
    """[n, d] un-normalised N(0, sigma^2) rows (norms far from 1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (sigma * rng.standard_normal((n, d))).astype(dtype)


def sample_rows(n: int, k: int, seed: int) -> np.ndarray:
    """k distinct row indices of [0, n), sorted (oracle row sample for the
    large configs; independent of the device layout)."""
    rng = np.random.default_rng(seed ^ 0x5A)
    k = min(k, n)
    return np.sort(rng.choice(n, size=k, replace=False))


def chunk_seed(seed: int, chunk: int) -> int:
    """64-bit seed of chunk ``chunk`` of the batch with base seed ``seed``."""
    st = np.random.SeedSequence([int(seed), int(chunk)]).generate_state(2, np.uint32)
    return int(st[0]) | (int(st[1]) << 32)


def device_unit_vectors(n: int, d: int, seed: int, torch_dtype, device, chunk_rows: int = CHUNK_ROWS,
                        row0: int = 0):
    """Device-resident isotropic unit vectors for the large configs: global
    rows [row0, row0 + n) of the batch with base seed ``seed``.  Chunk c
    (global rows [c*chunk_rows, (c+1)*chunk_rows)) is drawn whole with torch's
    generator seeded chunk_seed(seed, c), normalised in fp32 and cast, so a
    shard of the batch equals the same rows of the whole batch.  Returns a
    contiguous [n, d] tensor."""
    import torch
    out = torch.empty((n, d), dtype=torch_dtype, device=device)
    gen = torch.Generator(device=device)
    r = row0
    while r < row0 + n:
        c = r // chunk_rows
        lo, hi = c * chunk_rows, (c + 1) * chunk_rows
        take_hi = min(hi, row0 + n)
        gen.manual_seed(chunk_seed(seed, c))
        # always the whole chunk (the generator's output for a shorter draw
        # is not a prefix of the longer one), then the rows wanted
        g = torch.randn((chunk_rows, d), generator=gen, device=device, dtype=torch.float32)[r - lo:take_hi - lo]
        g = g / g.norm(dim=1, keepdim=True).clamp_min(1e-30)
        out[r - row0:take_hi - row0].copy_(g.to(torch_dtype))
        r = take_hi
    return out
