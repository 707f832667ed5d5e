"""Seeded problem builders shared by the parity tests (and the smoke test)."""
from __future__ import annotations

import numpy as np

from paper_2103_11050_b200 import api


def random_kappa(nx, ny, seed, lo=0.3, hi=3.0):
    """log-uniform kappa in [lo, hi] (the reference tests' random_kappa, test_mrcm.cpp:21-28)."""
    rng = np.random.default_rng(seed)
    return np.exp(rng.uniform(np.log(lo), np.log(hi), nx * ny))


def problem(nx, ny, nsx, nsy, K, bc=None, lx=1.0, ly=1.0, M=5.0, q=None, space=api.SPACE_CONSTANT,
            hbar=api.HBAR_WHOLE, alpha=None):
    bc = bc if bc is not None else api.pressure_drop(nx, ny)
    return api.Problem(nx, ny, lx, ly, nsx, nsy, np.asarray(K, np.float64), bc, viscosity_ratio=M, q=q,
                       space_kind=space, hbar_mode=hbar, alpha=alpha or api.AlphaSpec())


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)
