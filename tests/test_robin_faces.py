"""Physical Robin faces (FaceBc::robin, proj/include/mrcmflow/elliptic.hpp:16-28):
-beta u.n_out + p_face = robin_rhs on an exterior face.

The reference assembles them in CellCenteredSolver (elliptic.cpp:133-136,
176-177, 231-235), copies them through restrict_physical_data
(mrcm.cpp:121-123), keeps their data in the homogeneous problems (only
non-Robin values are zeroed, mrcm.cpp:166-167) and in the MPM-2P delta problem
(mpm.cpp:80-81), and counts them neither as pure-Neumann nor as grounding
faces (elliptic.hpp:46-50, mrcm.cpp:333-336).

CPU part: the oracle against the exact 1-D answer. GPU part: the CUDA path
against the oracle (mrcm_solve, mpm_pressure_update, the fine solve and a
short run).
"""
import numpy as np
import pytest

from cases import problem, random_kappa, rel_l2
from paper_2103_11050_b200 import api

TOL_PU = 1e-8
TOL_S = 1e-8


def robin_slab(nx, ny, beta, rhs, g_east=0.0):
    """Robin on the west side, p = g_east on the east, no flow on south/north."""
    return api.BoundarySpec.uniform(nx, ny, (api.ROBIN, beta, rhs), (api.PRESSURE, g_east), (api.FLUX, 0.0),
                                    (api.FLUX, 0.0))


def exact_slab(nx, ny, beta, rhs, g_east=0.0):
    """K = 1 on the unit square: p(x) = a (x - 1) + g_east with
    -beta u.n_out + p(0) = rhs, u.n_out = a at x = 0 (outward normal -x,
    u = -a), so -beta a - a + g_east = rhs. TPFA with half-cell boundary
    transmissibilities is exact for linear p."""
    a = (g_east - rhs) / (1.0 + beta)
    xc = (np.arange(nx) + 0.5) / nx
    p = np.tile(a * (xc - 1.0) + g_east, ny)
    return p, -a


def test_oracle_robin_slab_exact(oracle):
    nx, ny, beta, rhs = 24, 8, 0.7, 2.0
    prob = problem(nx, ny, 1, 1, np.ones(nx * ny), bc=robin_slab(nx, ny, beta, rhs))
    o = api.Simulator(prob, oracle)
    p_ex, u_ex = exact_slab(nx, ny, beta, rhs)
    p, u = o.fine_solve(np.ones(nx * ny))
    assert np.max(np.abs(p - p_ex)) < 1e-12
    assert np.max(np.abs(u[:(nx + 1) * ny] - u_ex)) < 1e-12
    # The multiscale solve is exact too (vertical interfaces only: p and the flux are constant along each
    # one) when the Robin face carries no data: the reference's
    # homogeneous problems keep a physical Robin face's robin_rhs
    # (mrcm.cpp:166-167), so with robin_rhs != 0 each basis function carries
    # it as well and the recombined MRCM answer is not the exact one — a
    # property of the reference that the oracle and the GPU path reproduce.
    p_ex0, u_ex0 = exact_slab(nx, ny, beta, 0.0, 1.0)
    prob4 = problem(nx, ny, 4, 1, np.ones(nx * ny), bc=robin_slab(nx, ny, beta, 0.0, 1.0))
    s = api.Simulator(prob4, oracle).mrcm_solve(np.ones(nx * ny))
    assert np.max(np.abs(s.p - p_ex0)) < 1e-10
    assert np.max(np.abs(s.u[:(nx + 1) * ny] - u_ex0)) < 1e-10


def test_robin_requires_positive_beta(oracle):
    nx = ny = 8
    prob = problem(nx, ny, 2, 2, np.ones(nx * ny), bc=robin_slab(nx, ny, 0.0, 1.0))
    with pytest.raises(api.ConfigError):
        api.Simulator(prob, oracle).mrcm_solve(np.ones(nx * ny))


def _bcs(nx, ny):
    return {
        "robin_west": robin_slab(nx, ny, 0.4, 1.5),
        "robin_all": api.BoundarySpec.uniform(nx, ny, (api.ROBIN, 0.5, 1.0), (api.ROBIN, 2.0, -0.5),
                                              (api.ROBIN, 1.0, 0.25), (api.ROBIN, 0.3, 0.0)),
        "robin_mixed": api.BoundarySpec.uniform(nx, ny, (api.FLUX, -1.0), (api.ROBIN, 0.8, 0.0), (api.FLUX, 0.0),
                                                (api.ROBIN, 1.2, 0.3)),
    }


@pytest.mark.gpu
@pytest.mark.parametrize("bcn", ["robin_west", "robin_all", "robin_mixed"])
@pytest.mark.parametrize("nsx,nsy,space", [(4, 4, api.SPACE_CONSTANT), (3, 2, api.SPACE_LINEAR), (2, 1, api.SPACE_CONSTANT)])
def test_robin_mrcm_mpm_fine_parity(oracle, bcn, nsx, nsy, space):
    nx, ny = 48, 32
    K = random_kappa(nx, ny, 21, 0.1, 10.0)
    prob = problem(nx, ny, nsx, nsy, K, bc=_bcs(nx, ny)[bcn], space=space)
    g, o = api.Simulator(prob), api.Simulator(prob, oracle)
    sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
    assert sg.counters == so.counters
    assert rel_l2(sg.p, so.p) < TOL_PU and rel_l2(sg.u, so.u) < TOL_PU
    rng = np.random.default_rng(4)
    for amp in (0.0, 0.1):
        kn = K * np.exp(amp * rng.standard_normal(K.size))
        mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
        assert mg.counters == mo.counters
        assert rel_l2(mg.p, mo.p) < TOL_PU and rel_l2(mg.u, mo.u) < TOL_PU
    pg, ug = g.fine_solve(K)
    po, uo = o.fine_solve(K)
    assert rel_l2(pg, po) < TOL_PU and rel_l2(ug, uo) < TOL_PU


@pytest.mark.gpu
def test_robin_slab_exact_on_device():
    nx, ny, beta = 64, 32, 0.7
    p_ex, u_ex = exact_slab(nx, ny, beta, 0.0, 1.0)
    g = api.Simulator(problem(nx, ny, 4, 1, np.ones(nx * ny), bc=robin_slab(nx, ny, beta, 0.0, 1.0)))
    s = g.mrcm_solve(np.ones(nx * ny))
    assert np.max(np.abs(s.p - p_ex)) < 1e-10
    assert np.max(np.abs(s.u[:(nx + 1) * ny] - u_ex)) < 1e-10
    p, u = g.fine_solve(np.ones(nx * ny))
    assert np.max(np.abs(p - p_ex)) < 1e-10


@pytest.mark.gpu
def test_robin_run_parity(oracle):
    nx = ny = 64
    K = random_kappa(nx, ny, 8, 0.1, 10.0)
    bc = api.BoundarySpec.uniform(nx, ny, (api.ROBIN, 0.5, 1.0), (api.PRESSURE, 0.0), (api.FLUX, 0.0),
                                  (api.FLUX, 0.0))
    prob = problem(nx, ny, 4, 4, K, bc=bc, M=5.0)
    sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, te=60, cfl_safety=0.5)
    rg, ro = api.Simulator(prob).run(sp), api.Simulator(prob, oracle).run(sp)
    assert [s["rebuilt"] for s in rg.record.steps] == [s["rebuilt"] for s in ro.record.steps]
    assert rg.record.counters == ro.record.counters
    assert np.max(np.abs(rg.s_final - ro.s_final)) <= TOL_S
    assert rel_l2(rg.p_final, ro.p_final) <= TOL_PU and rel_l2(rg.u_final, ro.u_final) <= TOL_PU


@pytest.mark.parametrize("gpu", [False, pytest.param(True, marks=pytest.mark.gpu)])
def test_pure_flux_multisubdomain_is_singular(oracle, gpu):
    """No Pressure or Robin face and more than one subdomain: the interface
    system inherits the constant null space, and the reference's rcond guard
    raises NumericError (mrcm.cpp:227-238). Robin faces ground the pressure
    without grounding the repair (robin_all above: the repair then pins
    subdomain 0, mrcm.cpp:360-367)."""
    nx, ny = 48, 32
    K = random_kappa(nx, ny, 5, 0.1, 10.0)
    bc = api.BoundarySpec.uniform(nx, ny, (api.FLUX, -1.0), (api.FLUX, 1.0), (api.FLUX, 0.0), (api.FLUX, 0.0))
    sim = api.Simulator(problem(nx, ny, 4, 4, K, bc=bc), None if gpu else oracle)
    with pytest.raises(api.NumericError):
        sim.mrcm_solve(K)
