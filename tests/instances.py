"""Seeded random assembly instances for the parity corpus.

Restates the recipe of the reference's test fixture ``random_instance``
(/root/reference/pkg/tests/conftest.py:32-57) so the same seeds give the same
triplets without the reference present: log-uniform length in [0, max_len],
5% empty instances, a quarter with tiny dimensions 1..7 (near-total
collision, long duplicate runs), otherwise dimensions up to max_dim; values
N(0,1), 30% of instances with 5% exact zeros, 15% with 5% NaNs.
tests/golden/sweep_digests.json pins that the restatement reproduces the
reference's inputs bit for bit (input digests) and holds the reference's
outputs (output digests).
"""

from __future__ import annotations

import hashlib

import numpy as np


def random_triplets(seed, max_len=50_000, max_dim=2000, allow_special=True):
    """Returns (ii int64, jj int64, sr float64); dims are inferred (max index)."""
    rng = np.random.default_rng(seed)
    length = int(np.expm1(rng.uniform(0, np.log1p(max_len))))
    if rng.random() < 0.05:
        length = 0
    if rng.random() < 0.25:
        m = int(rng.integers(1, 8))
        n = int(rng.integers(1, 8))
    else:
        m = int(rng.integers(1, max_dim + 1))
        n = int(rng.integers(1, max_dim + 1))
    ii = rng.integers(1, m + 1, size=length)
    jj = rng.integers(1, n + 1, size=length)
    sr = rng.standard_normal(length)
    if allow_special and length:
        if rng.random() < 0.3:
            sr[rng.integers(0, length, size=max(1, length // 20))] = 0.0
        if rng.random() < 0.15:
            sr[rng.integers(0, length, size=max(1, length // 20))] = np.nan
    return ii, jj, sr


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()[:32]


def input_digest(ii, jj, sr) -> str:
    return digest(np.asarray(ii, dtype=np.int32), np.asarray(jj, dtype=np.int32),
                  np.asarray(sr, dtype=np.float64))


def output_digest(jc, ir, pr) -> str:
    return digest(np.asarray(jc, dtype=np.int32), np.asarray(ir, dtype=np.int32),
                  np.asarray(pr, dtype=np.float64))


SWEEP_SEED_BASE = 1_000_000
SWEEP_COUNT = 1000
