"""Richer interface spaces on the BASELINE.json fields: the
cases tools/make_space_fixtures.py runs through the oracle and
tests/test_gpu_spaces.py through the GPU.

Each case: the config's field, boundary spec and fluid, with the interface
space swapped; a short run (te elliptic solves) with the config's splitting
policy, or MRCM every step where the case exists to exercise rebuilds."""
from __future__ import annotations

import dataclasses

from paper_2103_11050_b200 import api, configs

EDGE = dict(hbar_mode=api.HBAR_PER_EDGE)
LIN_ADAPT = dict(space_kind=api.SPACE_LINEAR, alpha=api.AlphaSpec(mode=api.ALPHA_ADAPTIVE))
LIN = dict(space_kind=api.SPACE_LINEAR)
ADAPT = dict(alpha=api.AlphaSpec(mode=api.ALPHA_ADAPTIVE))
HALF = dict(hbar_mode=api.HBAR_HALF)

# name: (config, space knobs, te, method override, full fields?, banded oracle interface LU?)
CASES = {
    # C2 per-edge: 256 subdomains of 16x16, 128 homogeneous solves each,
    # interface dim 15,360 (dense path on the GPU); 21 steps, 6 rebuilds
    "C2_edge": ("C2", EDGE, 21, None, True, True),
    # C2 with the high-contrast preset's space: linear + adaptive alpha
    "C2_linad": ("C2", LIN_ADAPT, 61, None, True, False),
    # C4 per-edge: 256 subdomains of 32x32, 256 homogeneous solves each,
    # interface dim 30,720 (block cyclic reduction on the GPU); MRCM every step
    "C4_edge": ("C4", EDGE, 4, api.MRCM_EVERY_STEP, True, True),
    "C4_linad": ("C4", LIN_ADAPT, 21, None, True, False),
    # C5 (16,384 subdomains): linear space (dim 130,048), adaptive alpha, half
    # segments; the initial MRCM solve and three MPM-2P updates
    "C5_lin": ("C5", LIN, 4, None, False, True),
    "C5_adapt": ("C5", ADAPT, 4, None, False, True),
    "C5_half": ("C5", HALF, 4, None, False, True),
}


def build_case(name):
    cfg_name, knobs, te, method, full, banded = CASES[name]
    cfg = configs.build(cfg_name)
    prob = dataclasses.replace(cfg.problem, **knobs)
    split = dataclasses.replace(cfg.split, te=te, stop_on_breakthrough=False)
    if method is not None:
        split = dataclasses.replace(split, method=method)
    return prob, split, cfg.s0(), full, banded
