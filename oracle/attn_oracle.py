"""Fused KV-cache decode consumer, CPU ORACLE (fp64, NumPy) — TEST
INFRASTRUCTURE ONLY (same rules as ``iq_oracle``).

What the consumer computes (R25-R27; "attention-logit
preservation and inner-product error under the complete two-stage
pipeline"): the attention logit of query q against every cached key, from
the key's codes alone,

    s[j, k] = <q_j, x^_k>                                   (stage 1, R25)
            + sqrt(pi/2)/m * gamma_k * <S q_j, sign_k>      (stage 2, R24)

written as its plain definition: decode every key with Algorithm 1's decoder
(``iq_oracle.decode``) and take the dot products.  The kernel's route (rotate
the query, <q, T^-1 c> = <T q, c>) is NOT used here; tests/test_oracle_attn.py
pins the two against each other and against brute-force loops.
"""
from __future__ import annotations

import math

import numpy as np

from . import iq_oracle as O


def attention_scores(Q, codes, rho, p: O.OracleParams, q01=None, gamma=None, S=None) -> np.ndarray:
    """Q [n_q, d]; codes [n_keys, padded d] (unpacked); rho [n_keys].
    Returns scores [n_q, n_keys] in fp64."""
    Q = np.asarray(Q, dtype=np.float64)
    xh = O.decode(codes, np.asarray(rho, dtype=np.float64), p)       # [n_keys, d]
    s = Q @ xh.T
    if q01 is not None:
        m = S.shape[0]
        sign = 2.0 * np.asarray(q01, dtype=np.float64) - 1.0           # [n_keys, m]
        s = s + (math.sqrt(math.pi / 2.0) / m) * np.asarray(gamma, dtype=np.float64)[None, :] * ((Q @ S.T) @ sign.T)
    return s
