"""Helpers shared by tools/make_fixtures.py (writes the oracle fixtures) and
the GPU parity tests (read them): mantissa rounding of stored fields and the
seeded random-projection sketch used for C5's 16.8 M-cell fields."""
from __future__ import annotations

import numpy as np

N_SKETCH = 64
SKETCH_SEED = 20260


def round_mantissa(x, bits=32):
    """float64 with the low (52 - bits) mantissa bits cleared (round to nearest)."""
    v = np.ascontiguousarray(x, np.float64).view(np.uint64)
    drop = np.uint64(52 - bits)
    half = np.uint64(1) << (drop - np.uint64(1))
    r = ((v + half) >> drop) << drop
    return r.view(np.float64)


def rademacher(n, k, seed=SKETCH_SEED):
    """Row k of the sketch matrix: n seeded +-1 values (float64)."""
    rng = np.random.default_rng([seed, k, n])
    return rng.integers(0, 2, n, dtype=np.int8).astype(np.float64) * 2.0 - 1.0


def sketch(x, n_sketch=N_SKETCH):
    """64 Rademacher projections: for a difference d, mean_k (r_k.d)^2 estimates |d|^2."""
    return np.array([rademacher(x.size, k) @ x for k in range(n_sketch)])


def subsample_idx(n, frac=256, seed=SKETCH_SEED):
    rng = np.random.default_rng([seed, 7, n])
    return np.sort(rng.choice(n, size=max(1, n // frac), replace=False))
