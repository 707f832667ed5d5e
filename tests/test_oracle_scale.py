"""The oracle features that make C5 and C3 checkable (CPU only).

* Banded partial-pivot LU of the interface matrix (the C5 path: the
  reference's dense PartialPivLU, mrcm.cpp:198,226-238, would need 34 GB):
  the same M entries bit for bit, the same solution to roundoff, the same
  rcond > 1e-14 guard, on the decompositions and spaces of the parity cases.
* Per-subdomain threading: bit-identical results.
* The long-double build: agrees with the double build to roundoff on a
  well-conditioned case (it is the exact-answer yardstick for C3).
* The committed full-run fixtures are self-consistent (counter ledger).
"""
import os

import numpy as np
import pytest

from cases import problem, random_kappa, rel_l2
from paper_2103_11050_b200 import api, configs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = [(32, 32, 4, 4, api.SPACE_CONSTANT, api.HBAR_WHOLE), (32, 32, 4, 4, api.SPACE_LINEAR, api.HBAR_WHOLE),
         (16, 16, 2, 2, api.SPACE_CONSTANT, api.HBAR_PER_EDGE), (48, 32, 6, 2, api.SPACE_CONSTANT, api.HBAR_HALF),
         (60, 40, 3, 2, api.SPACE_CONSTANT, api.HBAR_WHOLE), (16, 8, 4, 1, api.SPACE_CONSTANT, api.HBAR_WHOLE)]


@pytest.fixture
def solver_mode(oracle):
    def set_mode(m):
        oracle.dll.oracle_set_interface_solver(m)
    yield set_mode
    oracle.dll.oracle_set_interface_solver(0)


@pytest.mark.parametrize("case", CASES)
def test_banded_interface_lu_matches_dense(oracle, solver_mode, case):
    nx, ny, nsx, nsy, space, hbar = case
    K = random_kappa(nx, ny, 11, 0.01, 100.0)
    prob = problem(nx, ny, nsx, nsy, K, space=space, hbar=hbar)
    out = []
    for mode in (1, 2):
        solver_mode(mode)
        s = api.Simulator(prob, oracle)
        g = s.mrcm_solve(K)
        M = s.interface_matrix()
        m = s.mpm_pressure_update(K * np.exp(0.05 * np.random.default_rng(1).standard_normal(K.size)))
        out.append((g, M, m))
        s.close()
    (gd, Md, md), (gb, Mb, mb) = out
    assert np.array_equal(Md, Mb)  # same entries, same accumulation order
    assert rel_l2(gb.coeffs, gd.coeffs) < 1e-12
    for a, b in ((gb.p, gd.p), (gb.u, gd.u), (mb.p, md.p), (mb.u, md.u)):
        assert rel_l2(a, b) < 1e-12


def test_banded_interface_lu_singular_guard(oracle, solver_mode):
    """All-Flux physical BCs make M singular: both solvers raise NumericError (mrcm.cpp:227-238)."""
    nx = ny = 32
    K = random_kappa(nx, ny, 3)
    bc = api.BoundarySpec.uniform(nx, ny, (api.FLUX, 0.0), (api.FLUX, 0.0), (api.FLUX, 0.0), (api.FLUX, 0.0))
    for mode in (1, 2):
        solver_mode(mode)
        with pytest.raises(api.NumericError):
            api.Simulator(problem(nx, ny, 4, 4, K, bc=bc), oracle).mrcm_solve(K)


def test_threaded_oracle_bitwise(oracle):
    c = configs.build("C2", te_override=21)
    r1 = api.Simulator(c.problem, oracle).run(c.split, c.s0())
    oracle.dll.oracle_set_threads(4)
    try:
        r4 = api.Simulator(c.problem, oracle).run(c.split, c.s0())
    finally:
        oracle.dll.oracle_set_threads(1)
    assert np.array_equal(r1.s_final, r4.s_final) and np.array_equal(r1.u_final, r4.u_final)
    assert np.array_equal(r1.p_final, r4.p_final) and r1.record.counters == r4.record.counters


def test_long_double_oracle_agrees_on_well_conditioned_run():
    from oracle_bind import oracle_lib
    c = configs.build("C1", te_override=41)
    rd = api.Simulator(c.problem, oracle_lib()).run(c.split, c.s0())
    rx = api.Simulator(c.problem, oracle_lib(extended=True)).run(c.split, c.s0())
    assert [s["rebuilt"] for s in rd.record.steps] == [s["rebuilt"] for s in rx.record.steps]
    assert np.max(np.abs(rd.s_final - rx.s_final)) < 1e-11
    assert rel_l2(rd.u_final, rx.u_final) < 1e-12 and rel_l2(rd.p_final, rx.p_final) < 1e-12


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_fixture_ledger(name):
    """Counters of each committed full-run fixture reconcile with its decision
    sequence (test_simulation.cpp:150-157): one interface solve per velocity
    update, N particular + N downscale per update, N-hat homogeneous per MRCM solve."""
    path = os.path.join(GOLDEN, f"run_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    fx = np.load(path)
    te, tm_total, tm_updates, bt, hom, part, down, fine, iface = fx["meta_int"][:9]
    reb = fx["rebuilt"]
    assert reb.size == te and reb[0] == 1 and int(reb.sum()) == tm_total and tm_updates == tm_total - 1
    assert iface == te and fine == 0 and part == down
    c = configs.build(name)
    n_sub = c.problem.nsx * c.problem.nsy
    assert down == te * n_sub
    assert hom % tm_total == 0
    assert np.all(np.diff(fx["bf_homog_cum"]) >= 0) and fx["bf_homog_cum"][-1] == hom
