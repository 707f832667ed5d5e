"""Richer interface spaces at scale against the oracle.

The BASELINE configs use the constant space with H-bar = H; the reference
also offers the per-edge space (H-bar = h), linear spaces and adaptive alpha
(proj/src/interface_space.cpp:9-52, proj/src/robin.cpp:39-92, the
`high-contrast` preset proj/src/config.cpp:474-475). These tests run them on
the BASELINE fields (tests/space_cases.py) on the GPU and compare with
oracle fixtures written by tools/make_space_fixtures.py:

  C2_edge   per-edge, 128 homogeneous solves per subdomain, dim 15,360 (dense
            interface inverse), 21 steps with 6 rebuilds
  C2_linad  linear + adaptive alpha, 61 steps, 15 rebuilds
  C4_edge   per-edge at 32x32 subdomains, 256 homogeneous solves each, dim
            30,720 (block cyclic reduction), MRCM every step
  C4_linad  linear + adaptive alpha on C4
  C5_lin / C5_adapt / C5_half  16,384 subdomains: initial MRCM solve + 3
            MPM-2P updates (linear space: dim 130,048)

Same bar as the full runs: decisions and counters exact, dt / PVI and the
fields within 1e-8 (C5 fields through the sketch + subsample). Where a
fixture carries the long-double run (ld_*), a field may instead be at least as
close to the extended-precision answer as the double-precision oracle is
(check_fields_vs_truth, the C3 / C5 rule)."""
import os

import numpy as np
import pytest

from paper_2103_11050_b200 import api
from space_cases import CASES, build_case
from test_gpu_full_runs import check_fields, check_fields_vs_truth, check_record, check_sketched_vs_truth

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", list(CASES))
def test_space_matches_oracle(name):
    path = os.path.join(GOLDEN, f"space_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path}: run tools/make_space_fixtures.py {name}")
    fx = dict(np.load(path))
    prob, split, s0, full, _ = build_case(name)
    assert split.te == int(fx["split_te"][0])
    with api.Simulator(prob) as sim:
        r = sim.run(split, s0)
    check_record(r, fx)
    if full and "ld_u" in fx:  # oracle roundoff above the bar: the extended-precision yardstick
        errs = check_fields_vs_truth(r, fx)
        print(f"{name}: rebuilds {r.record.update_steps}, errors {errs}")
        return
    if full:
        ds, dp, du = check_fields(r, fx)
        print(f"{name}: rebuilds {r.record.update_steps}, max|ds| {ds:.2e}, p {dp:.2e}, u {du:.2e}")
        return
    errs = check_sketched_vs_truth(r, fx, fx if "ld_u_sketch" in fx else None, prefix="ld_")
    print(f"{name}: rebuilds {r.record.update_steps}, errors {errs}")
