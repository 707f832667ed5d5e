"""CUDA path vs the CPU oracle through the C ABI (needs a B200).

Bar (BASELINE.json north_star): decisions and indexing bit-exact; p and u
relative L2 <= 1e-8; saturation max-abs <= 1e-8 after the full run.
Transport and beta are checked bitwise (the kernels keep the reference's
operation order under --fmad=false).
"""
import dataclasses

import numpy as np
import pytest

from cases import problem, random_kappa, rel_l2
from paper_2103_11050_b200 import api, configs

pytestmark = pytest.mark.gpu

TOL_PU = 1e-8   # relative L2 for pressure and velocity
TOL_S = 1e-8    # max-abs for saturation


def pair(prob, oracle):
    return api.Simulator(prob), api.Simulator(prob, oracle)


def test_gpu_library_is_the_cuda_path():
    lib = api.product_lib()
    assert lib.path.endswith("libmpm2p_b200.so")


def test_transport_bitwise(oracle):
    nx, ny = 48, 40
    K = random_kappa(nx, ny, 1, 0.1, 10.0)
    g, o = pair(problem(nx, ny, 4, 4, K, M=7.0), oracle)
    u = o.mrcm_solve(K).u
    rng = np.random.default_rng(3)
    s = rng.uniform(0, 1, nx * ny)
    assert np.array_equal(g.conductivity(s), o.conductivity(s))
    assert g.max_fractional_flow_slope() == o.max_fractional_flow_slope()
    for safety in (0.5, 0.9):
        assert g.cfl_timestep(u, safety, 1.0) == o.cfl_timestep(u, safety, 1.0)
    assert g.cfl_timestep(np.zeros_like(u), 0.9, 1.0) == 1.0
    dt = o.cfl_timestep(u, 0.9, 1.0)
    for inflow in (1.0, 0.3):
        assert np.array_equal(g.upwind_step(s, inflow, u, dt), o.upwind_step(s, inflow, u, dt))
        # injection rate: same terms, tree-summed on the device (reported PVI clock, not a parity quantity)
        assert abs(g.injection_rate(u, inflow) - o.injection_rate(u, inflow)) <= 1e-14 * abs(o.injection_rate(u, inflow))
    assert g.max_outlet_saturation(s, u) == o.max_outlet_saturation(s, u)
    assert np.array_equal(g.divergence(u), o.divergence(u))
    kn = K * np.exp(0.1 * rng.standard_normal(K.size))
    for mode in (api.EPS_RELATIVE, api.EPS_ABSOLUTE):
        e_g, e_o = g.epsilon(kn, K, mode), o.epsilon(kn, K, mode)
        assert abs(e_g - e_o) <= 1e-14 * e_o


def test_cfl_violation_raises(oracle):
    nx = ny = 16
    g, o = pair(problem(nx, ny, 1, 1, np.ones(nx * ny), M=1.0), oracle)
    u = np.zeros(g.faces)
    u[:(nx + 1) * ny] = 1.0
    for sim in (g, o):
        with pytest.raises(api.NumericError):
            sim.upwind_step(np.zeros(nx * ny), 1.0, u, 1.0)


@pytest.mark.parametrize("alpha_mode", [api.ALPHA_UNIFORM, api.ALPHA_ADAPTIVE])
def test_beta_bitwise(oracle, alpha_mode):
    nx, ny = 16, 12
    K = np.where(np.arange(ny)[:, None] < 2, 1e4, np.where(np.arange(ny)[:, None] >= ny - 2, 1e-4, 1.0))
    K = (K * np.ones((ny, nx))).ravel()
    K *= np.exp(0.01 * np.random.default_rng(0).standard_normal(K.size))
    g, o = pair(problem(nx, ny, 4, 3, K, alpha=api.AlphaSpec(mode=alpha_mode)), oracle)
    for a, b in zip(g.compute_beta(K), o.compute_beta(K)):
        assert np.array_equal(a, b)


MRCM_CASES = [
    # nx, ny, nsx, nsy, space, hbar, bc, lx, kappa range, q
    (32, 32, 4, 4, api.SPACE_CONSTANT, api.HBAR_WHOLE, "pd", 1.0, (0.3, 3.0), False),
    (32, 32, 4, 4, api.SPACE_CONSTANT, api.HBAR_HALF, "pd", 1.0, (0.1, 10.0), False),
    (16, 16, 2, 2, api.SPACE_CONSTANT, api.HBAR_PER_EDGE, "pd", 1.0, (0.1, 10.0), False),
    (32, 32, 4, 4, api.SPACE_LINEAR, api.HBAR_WHOLE, "pd", 1.0, (1e-2, 1e2), False),
    (12, 6, 3, 2, api.SPACE_LINEAR, api.HBAR_WHOLE, "ui", 2.0, (1e-2, 1e2), True),
    (40, 20, 2, 2, api.SPACE_CONSTANT, api.HBAR_WHOLE, "ui", 2.0, (0.3, 3.0), True),
    (16, 8, 4, 1, api.SPACE_CONSTANT, api.HBAR_WHOLE, "pd", 1.0, (0.3, 3.0), False),
    (12, 10, 1, 1, api.SPACE_CONSTANT, api.HBAR_WHOLE, "pd", 1.0, (1e-2, 1e2), True),
    (64, 64, 2, 2, api.SPACE_CONSTANT, api.HBAR_WHOLE, "pd", 1.0, (0.1, 10.0), False),
    (60, 40, 3, 2, api.SPACE_CONSTANT, api.HBAR_WHOLE, "pd", 1.5, (1e-3, 1e3), False),
]


@pytest.mark.parametrize("case", MRCM_CASES)
def test_mrcm_and_mpm_parity(oracle, case):
    nx, ny, nsx, nsy, space, hbar, bcn, lx, (lo, hi), with_q = case
    K = random_kappa(nx, ny, 11, lo, hi)
    q = np.random.default_rng(9).uniform(-1, 1, nx * ny) if with_q else None
    if with_q and bcn == "pd":
        q = q - q.mean()
    bc = api.pressure_drop(nx, ny) if bcn == "pd" else api.unit_inflow(nx, ny)
    adaptive = api.AlphaSpec(mode=api.ALPHA_ADAPTIVE if space == api.SPACE_LINEAR else api.ALPHA_UNIFORM)
    prob = problem(nx, ny, nsx, nsy, K, bc=bc, lx=lx, q=q, space=space, hbar=hbar, alpha=adaptive)
    g, o = pair(prob, oracle)
    sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
    assert sg.counters == so.counters
    if g.dim:
        assert rel_l2(g.interface_matrix(), o.interface_matrix()) < 1e-12
        assert rel_l2(sg.coeffs, so.coeffs) < 1e-9
    assert rel_l2(sg.p, so.p) < TOL_PU and rel_l2(sg.u, so.u) < TOL_PU
    assert sg.info.repair_warning == so.info.repair_warning
    assert sg.info.div_residual <= 1e-10 * sg.info.div_scale
    rng = np.random.default_rng(5)
    for amp in (0.0, 0.02, 0.2):
        kn = K * np.exp(amp * rng.standard_normal(K.size))
        mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
        assert mg.counters == mo.counters
        assert rel_l2(mg.p, mo.p) < TOL_PU and rel_l2(mg.u, mo.u) < TOL_PU
        assert mg.info.div_residual <= 1e-10 * mg.info.div_scale


def test_mrcm_with_given_beta(oracle):
    nx = ny = 32
    K = random_kappa(nx, ny, 2)
    g, o = pair(problem(nx, ny, 4, 4, K), oracle)
    bm, bp, _ = o.compute_beta(K)
    sg, so = g.mrcm_solve(K, (2 * bm, 3 * bp)), o.mrcm_solve(K, (2 * bm, 3 * bp))
    assert rel_l2(sg.p, so.p) < TOL_PU and rel_l2(sg.u, so.u) < TOL_PU


def test_interface_matrix_reused_byte_identically(oracle):
    """test_mpm.cpp:177-197: an MPM step leaves the cached interface matrix untouched."""
    nx = ny = 32
    K = random_kappa(nx, ny, 3)
    g = api.Simulator(problem(nx, ny, 4, 4, K))
    g.mrcm_solve(K)
    M0 = g.interface_matrix().copy()
    g.mpm_pressure_update(K * 1.004)
    assert np.array_equal(M0, g.interface_matrix())


def run_floor(oracle, prob, split, s0=None):
    """Solver-roundoff floor of the reference answer itself: the oracle run
    with natural vs reversed elimination order (both exact direct solves)."""
    ra = api.Simulator(prob, oracle).run(split, s0)
    oracle.dll.oracle_set_elimination_order(1)
    try:
        rb = api.Simulator(prob, oracle).run(split, s0)
    finally:
        oracle.dll.oracle_set_elimination_order(0)
    assert [x["rebuilt"] for x in ra.record.steps] == [x["rebuilt"] for x in rb.record.steps]
    return {"s": float(np.max(np.abs(ra.s_final - rb.s_final))), "p": rel_l2(ra.p_final, rb.p_final),
            "u": rel_l2(ra.u_final, rb.u_final)}


def _compare_runs(rg, ro, floor=None):
    floor = floor or {"s": 0.0, "p": 0.0, "u": 0.0}
    seq_g = [s["rebuilt"] for s in rg.record.steps]
    seq_o = [s["rebuilt"] for s in ro.record.steps]
    assert seq_g == seq_o
    assert rg.record.te == ro.record.te and rg.record.tm_total == ro.record.tm_total
    c_g, c_o = rg.record.counters, ro.record.counters
    assert (c_g.homogeneous, c_g.particular, c_g.downscale, c_g.interface_solves) == \
           (c_o.homogeneous, c_o.particular, c_o.downscale, c_o.interface_solves)
    assert rg.record.breakthrough_step == ro.record.breakthrough_step
    assert np.max(np.abs(rg.s_final - ro.s_final)) <= max(TOL_S, 10 * floor["s"])
    assert rel_l2(rg.p_final, ro.p_final) <= max(TOL_PU, 10 * floor["p"])
    assert rel_l2(rg.u_final, ro.u_final) <= max(TOL_PU, 10 * floor["u"])
    dts_g = np.array([s["dt"] for s in rg.record.steps])
    dts_o = np.array([s["dt"] for s in ro.record.steps])
    np.testing.assert_allclose(dts_g, dts_o, rtol=max(1e-8, 10 * floor["u"]))


@pytest.mark.parametrize("meth,mode,eta", [(api.MPM2P, api.EPS_RELATIVE, 0.01), (api.MPM2P, api.EPS_MOBILITY, 0.01),
                                           (api.MRCM_EVERY_STEP, api.EPS_RELATIVE, 0.01),
                                           (api.MPM2P_NO_UPDATES, api.EPS_RELATIVE, 0.01),
                                           (api.MPM2P, api.EPS_ABSOLUTE, 0.05), (api.MPM2P, api.EPS_RELATIVE, 0.0)])
def test_run_parity_small(oracle, meth, mode, eta):
    nx = ny = 64
    K = random_kappa(nx, ny, 7, 0.1, 10.0)
    g, o = pair(problem(nx, ny, 4, 4, K, M=5.0), oracle)
    sp = api.SplittingConfig(method=meth, eta=eta, eta_mode=mode, te=80, cfl_safety=0.5)
    _compare_runs(g.run(sp), o.run(sp))


def test_config_c1_full_run(oracle):
    """C1 (BASELINE configs[0]) end to end: 200 saturation steps."""
    c = configs.build("C1")
    g, o = pair(c.problem, oracle)
    rg, ro = g.run(c.split, c.s0()), o.run(c.split, c.s0())
    _compare_runs(rg, ro)
    assert rg.record.max_div_ratio <= 1e-10


def test_config_c3_two_pass(oracle):
    """C3: run to breakthrough, then to breakthrough + 50% (bounded here by max_steps_hard)."""
    import dataclasses
    c = configs.build("C3")
    sp = dataclasses.replace(c.split, max_steps_hard=400)
    g, o = pair(c.problem, oracle)
    r1g, r1o = g.run(sp, c.s0()), o.run(sp, c.s0())
    # C3's field spans 1.6e7 in K (cond(M) ~ 2e9): the reference's own direct
    # solves carry ~1e-7 roundoff in u, measured here as the floor.
    _compare_runs(r1g, r1o, run_floor(oracle, c.problem, sp, c.s0()))
    if r1g.record.breakthrough_step >= 0:
        te = configs.breakthrough_plus_50(r1g.record.breakthrough_step)
        sp2 = dataclasses.replace(sp, stop_on_breakthrough=False, te=min(te, 400))
        _compare_runs(g.run(sp2, c.s0()), o.run(sp2, c.s0()), run_floor(oracle, c.problem, sp2, c.s0()))


@pytest.mark.parametrize("name,steps", [("C2", 120), ("C4", 40)])
def test_config_samples(oracle, name, steps):
    """Bounded samples of C2 / C4 (full runs are benched, not oracle-checked)."""
    c = configs.build(name, te_override=steps + 1)
    g, o = pair(c.problem, oracle)
    _compare_runs(g.run(c.split, c.s0()), o.run(c.split, c.s0()))


def test_determinism_and_eta0_equivalence():
    """test_simulation.cpp:95-120: bitwise-identical reruns; eta = 0 == rebuild every step."""
    c = configs.build("C1", te_override=40)
    g = api.Simulator(c.problem)
    a, b = g.run(c.split, c.s0()), g.run(c.split, c.s0())
    assert np.array_equal(a.s_final, b.s_final) and np.array_equal(a.u_final, b.u_final)
    assert [s["epsilon"] for s in a.record.steps] == [s["epsilon"] for s in b.record.steps]
    import dataclasses
    e0 = g.run(dataclasses.replace(c.split, eta=0.0), c.s0())
    ev = g.run(dataclasses.replace(c.split, method=api.MRCM_EVERY_STEP), c.s0())
    assert np.array_equal(e0.s_final, ev.s_final)
    assert [s["rebuilt"] for s in e0.record.steps] == [1] * len(e0.record.steps)


def test_full_size_properties_c2():
    """At C2's full size: conservative velocities, saturation in [0,1], and a
    zero-perturbation MPM update reproduces the MRCM solution."""
    c = configs.build("C2", te_override=60)
    g = api.Simulator(c.problem)
    r = g.run(c.split, c.s0())
    assert r.record.max_div_ratio <= 1e-10
    assert r.s_final.min() >= 0.0 and r.s_final.max() <= 1.0
    K = c.problem.K
    sol = g.mrcm_solve(K)
    m = g.mpm_pressure_update(K)
    assert rel_l2(m.u, sol.u) < 1e-10 and rel_l2(m.p, sol.p) < 1e-10


def test_config_errors():
    nx = ny = 16
    with pytest.raises(api.ConfigError):
        api.Simulator(problem(nx, ny, 3, 3, np.ones(nx * ny)))
    g = api.Simulator(problem(nx, ny, 2, 2, np.ones(nx * ny)))
    with pytest.raises(api.ConfigError):
        g.run(api.SplittingConfig(te=0))
    # the fine-reference method runs on the device (fine.cu): one fine solve per velocity update
    assert g.run(api.SplittingConfig(te=3, method=api.FINE_REFERENCE)).record.counters.fine == 3
    with pytest.raises(api.ConfigError):
        g.mpm_pressure_update(np.ones(nx * ny))
    bad = np.ones(nx * ny)
    bad[3] = -1.0
    with pytest.raises(api.NumericError):
        g.mrcm_solve(bad)


# ---- K7: MINRES interface solve (the path C5 takes; forced here at small sizes)

def _krylov_sim(prob):
    import os
    os.environ["MPM2P_IFACE"] = "krylov"
    try:
        return api.Simulator(prob)
    finally:
        os.environ.pop("MPM2P_IFACE", None)


@pytest.mark.parametrize("nsx,nsy,space,hbar,contrast", [(4, 4, api.SPACE_CONSTANT, api.HBAR_WHOLE, 10.0),
                                                         (4, 4, api.SPACE_LINEAR, api.HBAR_WHOLE, 10.0),
                                                         (2, 4, api.SPACE_CONSTANT, api.HBAR_HALF, 100.0),
                                                         (8, 8, api.SPACE_CONSTANT, api.HBAR_WHOLE, 1e3)])
def test_krylov_interface_parity(oracle, nsx, nsy, space, hbar, contrast):
    """MINRES on K = J M (quasi-definite) vs the reference's LU, through mrcm_solve and mpm_update."""
    nx = ny = 32
    K = random_kappa(nx, ny, 1, 1.0 / contrast, 1.0)
    prob = problem(nx, ny, nsx, nsy, K, M=5.0, space=space, hbar=hbar)
    g, o = _krylov_sim(prob), api.Simulator(prob, oracle)
    sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
    assert sg.counters == so.counters
    assert rel_l2(g.interface_matrix(), o.interface_matrix()) < 1e-12  # scattered from the CSR operator
    for a, b in ((sg.coeffs, so.coeffs), (sg.p, so.p), (sg.u, so.u)):
        assert rel_l2(a, b) <= 1e-10
    kn = K * np.exp(0.05 * np.random.default_rng(3).standard_normal(K.size))
    mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
    assert rel_l2(mg.p, mo.p) <= 1e-10 and rel_l2(mg.u, mo.u) <= 1e-10


def test_krylov_matches_dense_c1_run():
    """A whole C1 run with the MINRES interface solve vs the dense-inverse path:
    same decisions, fields within roundoff."""
    c = configs.build("C1")
    rd = api.Simulator(c.problem).run(c.split, c.s0())
    rk = _krylov_sim(c.problem).run(c.split, c.s0())
    assert rk.record.interface_krylov == 1 and rd.record.interface_krylov == 0
    assert rk.record.interface_iterations > 0
    assert [s["rebuilt"] for s in rk.record.steps] == [s["rebuilt"] for s in rd.record.steps]
    assert np.max(np.abs(rk.s_final - rd.s_final)) <= TOL_S
    assert rel_l2(rk.p_final, rd.p_final) <= TOL_PU and rel_l2(rk.u_final, rd.u_final) <= TOL_PU


def test_c5_scale_properties():
    """C5 (128 x 128 subdomains, interface dim 65,024: beyond the dense path,
    solved by the block-tridiagonal direct solver) through size-independent
    properties: conservative
    velocities, saturation in [0, 1], the PVI clock advancing, counters of an
    Algorithm-1 run, and a zero-perturbation MPM update reproducing MRCM."""
    c = configs.build("C5", te_override=3)
    g = api.Simulator(c.problem)
    assert g.dim == 65024
    r = g.run(c.split, c.s0())
    rec = r.record
    assert rec.interface_krylov == 2  # direct block-tridiagonal (the dense inverse would be 34 GB)
    assert rec.max_div_ratio <= 1e-9
    assert r.s_final.min() >= 0.0 and r.s_final.max() <= 1.0 and r.s_final.max() > 0.0
    assert rec.final_pvi > 0.0 and rec.te == 3
    assert rec.counters.downscale % (128 * 128) == 0 and rec.counters.downscale >= (rec.te - 1) * 128 * 128
    K = c.problem.K
    sol = g.mrcm_solve(K)
    m = g.mpm_pressure_update(K)
    assert rel_l2(m.u, sol.u) < 1e-9 and rel_l2(m.p, sol.p) < 1e-9


def test_repeated_rebuilds_bitwise_stable(oracle):
    """Regression for a cross-sweep shared-memory race (a sweep's trailing
    cp.async prefetches landing in the next sweep's ring): many rebuilds of a
    64-subdomain, B = 4 system must give bit-identical interface matrices and
    solutions, equal to the oracle's within the parity bar."""
    nx = ny = 32
    K = random_kappa(nx, ny, 1, 1e-3, 1.0)
    prob = problem(nx, ny, 8, 8, K, M=5.0)
    g = api.Simulator(prob)
    ref = g.mrcm_solve(K)
    M0 = g.interface_matrix()
    for _ in range(12):
        s = g.mrcm_solve(K)
        assert np.array_equal(g.interface_matrix(), M0)
        assert np.array_equal(s.p, ref.p) and np.array_equal(s.u, ref.u)
        m = g.mpm_pressure_update(K * 1.01)
        assert np.isfinite(m.p).all()
    so = api.Simulator(prob, oracle).mrcm_solve(K)
    assert rel_l2(ref.p, so.p) <= TOL_PU and rel_l2(ref.u, so.u) <= TOL_PU


# ---- K7b: direct block-tridiagonal interface solve (C5's default; forced here)

def _sim_iface(prob, mode):
    import os
    os.environ["MPM2P_IFACE"] = mode
    try:
        return api.Simulator(prob)
    finally:
        os.environ.pop("MPM2P_IFACE", None)


@pytest.mark.parametrize("nsx,nsy,space,hbar,contrast", [(4, 4, api.SPACE_CONSTANT, api.HBAR_WHOLE, 10.0),
                                                         (4, 4, api.SPACE_LINEAR, api.HBAR_WHOLE, 10.0),
                                                         (2, 4, api.SPACE_CONSTANT, api.HBAR_HALF, 100.0),
                                                         (8, 8, api.SPACE_CONSTANT, api.HBAR_WHOLE, 1e3),
                                                         (4, 1, api.SPACE_CONSTANT, api.HBAR_WHOLE, 10.0)])
def test_blocktri_interface_parity(oracle, nsx, nsy, space, hbar, contrast):
    """Block LDL^T of K = J M by subdomain rows vs the reference's LU."""
    nx = ny = 32
    K = random_kappa(nx, ny, 1, 1.0 / contrast, 1.0)
    prob = problem(nx, ny, nsx, nsy, K, M=5.0, space=space, hbar=hbar)
    g, o = _sim_iface(prob, "blocktri"), api.Simulator(prob, oracle)
    sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
    assert sg.counters == so.counters
    for a, b in ((sg.coeffs, so.coeffs), (sg.p, so.p), (sg.u, so.u)):
        assert rel_l2(a, b) <= 1e-10
    kn = K * np.exp(0.05 * np.random.default_rng(3).standard_normal(K.size))
    mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
    assert rel_l2(mg.p, mo.p) <= 1e-10 and rel_l2(mg.u, mo.u) <= 1e-10


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_blocktri_rcond_estimate(name):
    """The block-tridiagonal path's rcond guard (Hager/Higham with the block
    solves, as the oracle's banded path) against the dense path's exact
    1 / (||M||_1 ||M^-1||_1): the estimate of ||M^-1||_1 is a lower bound that
    is rarely off by more than a small factor."""
    c = configs.build(name, te_override=3)
    sp = dataclasses.replace(c.split, stop_on_breakthrough=False)
    rb = _sim_iface(c.problem, "blocktri").run(sp, c.s0(), c.inflow_sat)
    rd = _sim_iface(c.problem, "dense").run(sp, c.s0(), c.inflow_sat)
    exact, est = rd.record.min_rcond, rb.record.min_rcond
    assert rb.record.interface_krylov == 2 and exact > 0
    assert exact * (1 - 1e-9) <= est <= 10 * exact, (est, exact)


def test_blocktri_rcond_guard_raises():
    """Pure-flux data on several subdomains: the interface matrix is singular
    (constant null space). The block path now raises the reference's
    NumericError (mrcm.cpp:227-238) instead of returning garbage."""
    nx = ny = 32
    K = random_kappa(nx, ny, 5, 0.1, 10.0)
    bc = api.BoundarySpec.uniform(nx, ny, (api.FLUX, -1.0), (api.FLUX, 1.0), (api.FLUX, 0.0), (api.FLUX, 0.0))
    g = _sim_iface(problem(nx, ny, 4, 4, K, bc=bc), "blocktri")
    with pytest.raises(api.NumericError):
        g.mrcm_solve(K)


def test_blocktri_matches_dense_c2_sample():
    """A C2 sample run with the block-tridiagonal solve vs the dense inverse."""
    c = configs.build("C2", te_override=61)
    rd = api.Simulator(c.problem).run(c.split, c.s0())
    rb = _sim_iface(c.problem, "blocktri").run(c.split, c.s0())
    assert rb.record.interface_krylov == 2
    assert [s["rebuilt"] for s in rb.record.steps] == [s["rebuilt"] for s in rd.record.steps]
    assert np.max(np.abs(rb.s_final - rd.s_final)) <= TOL_S
    assert rel_l2(rb.p_final, rd.p_final) <= TOL_PU and rel_l2(rb.u_final, rd.u_final) <= TOL_PU


def _sim_env(prob, **env):
    """A context created with MPM2P_* switches set (read once, at creation)."""
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return api.Simulator(prob)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_split_downscale_matches_fused(oracle, name):
    """Split downscale (kappa_n operator factored on the side stream, sweeps on
    the critical path) vs the fused factor + solve: same decisions and
    counters, fields within the parity bar (C3: 10x its direct-solve floor)."""
    import dataclasses
    c = configs.build(name, te_override=41)
    split = dataclasses.replace(c.split, stop_on_breakthrough=False, te=41)
    rs = _sim_env(c.problem, MPM2P_DS_SPLIT=1).run(split, c.s0(), c.inflow_sat)
    rf = _sim_env(c.problem, MPM2P_DS_SPLIT=0).run(split, c.s0(), c.inflow_sat)
    assert [s["rebuilt"] for s in rs.record.steps] == [s["rebuilt"] for s in rf.record.steps]
    assert rs.record.counters == rf.record.counters
    fl = run_floor(oracle, c.problem, split, c.s0()) if name == "C3" else {"s": 0.0, "p": 0.0, "u": 0.0}
    assert np.max(np.abs(rs.s_final - rf.s_final)) <= max(TOL_S, 10 * fl["s"])
    assert rel_l2(rs.p_final, rf.p_final) <= max(TOL_PU, 10 * fl["p"])
    assert rel_l2(rs.u_final, rf.u_final) <= max(TOL_PU, 10 * fl["u"])


UPWIND_VARIANTS = {
    "col": dict(MPM2P_UPWIND_COL=1),
    "tile": dict(MPM2P_UPWIND_COL=0, MPM2P_UPWIND_TILE=1),
    "cell": dict(MPM2P_UPWIND_COL=0, MPM2P_UPWIND_TILE=0),
}


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_upwind_variants_bitwise(name):
    """Column-marching, tiled and one-thread-per-cell upwind steps give
    bit-identical saturation, dt sequence and clamp counts over a run."""
    c = configs.build(name, te_override=31)
    runs = {k: _sim_env(c.problem, **env).run(c.split, c.s0(), c.inflow_sat) for k, env in UPWIND_VARIANTS.items()}
    a = runs["col"]
    for k in ("tile", "cell"):
        b = runs[k]
        assert np.array_equal(a.s_final, b.s_final) and np.array_equal(a.u_final, b.u_final), k
        assert [s["dt"] for s in a.record.steps] == [s["dt"] for s in b.record.steps], k
        assert a.record.clamp_count == b.record.clamp_count, k


@pytest.mark.parametrize("variant", sorted(UPWIND_VARIANTS))
@pytest.mark.parametrize("nx,ny,sx,sy", [(31, 7, 1, 1), (62, 45, 2, 3), (93, 130, 3, 5), (300, 20, 10, 1),
                                         (256, 256, 16, 16)])
def test_upwind_step_ragged_bitwise(oracle, variant, nx, ny, sx, sy):
    """upwind_step on widths that are not multiples of a warp's 30 columns or a
    tile, heights that end mid row-chunk, and a velocity field with both signs
    on every face family, bit-identical to the oracle (transport.cpp:73-120)."""
    rng = np.random.default_rng(nx * 1000 + ny)
    prob = problem(nx, ny, sx, sy, np.ones(nx * ny), M=3.0)
    g = _sim_env(prob, **UPWIND_VARIANTS[variant])
    o = api.Simulator(prob, oracle)
    u = rng.standard_normal(g.faces)
    s = rng.uniform(0.05, 0.95, nx * ny)
    dt = 0.02 * o.cfl_timestep(u, 0.9, 1.0)  # random u is not divergence-free: keep s inside [0, 1]
    for inflow in (1.0, 0.25):
        assert np.array_equal(g.upwind_step(s, inflow, u, dt), o.upwind_step(s, inflow, u, dt))


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_kappa_col_bitwise(name):
    """Row-marching k_kappa_col vs one thread per cell: kappa and the fused
    transmissibilities are bit-identical, so whole runs are (the drift sums
    only change their partition into double-double partials)."""
    c = configs.build(name, te_override=31)
    a = _sim_env(c.problem, MPM2P_KAPPA_COL=1).run(c.split, c.s0(), c.inflow_sat)
    b = _sim_env(c.problem, MPM2P_KAPPA_COL=0).run(c.split, c.s0(), c.inflow_sat)
    assert [s["rebuilt"] for s in a.record.steps] == [s["rebuilt"] for s in b.record.steps]
    assert a.record.counters == b.record.counters and a.record.clamp_count == b.record.clamp_count
    for x, y in ((a.s_final, b.s_final), (a.p_final, b.p_final), (a.u_final, b.u_final)):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("nx,ny,sx,sy", [(31, 7, 1, 1), (62, 45, 2, 3), (93, 130, 3, 5)])
def test_conductivity_col_ragged_bitwise(oracle, nx, ny, sx, sy):
    """conductivity through k_kappa_col on ragged sizes, bit-identical to the oracle."""
    rng = np.random.default_rng(nx + ny)
    K = np.exp(rng.standard_normal(nx * ny))
    prob = problem(nx, ny, sx, sy, K, M=4.0)
    g = _sim_env(prob, MPM2P_KAPPA_COL=1)
    o = api.Simulator(prob, oracle)
    s = rng.uniform(0.0, 1.0, nx * ny)
    assert np.array_equal(g.conductivity(s), o.conductivity(s))


@pytest.mark.parametrize("nx,ny,nsx,nsy", [(32, 32, 4, 4), (48, 32, 6, 2), (64, 64, 16, 8)])
def test_separable_repair_parity(oracle, nx, ny, nsx, nsy):
    """The separable repair solve (Kronecker-sum eigen-decomposition, used
    above 4,096 subdomains) forced on small pressure-drop problems: vs the
    dense-inverse path and vs the oracle's dense LDL^T (mrcm.cpp:347-383)."""
    K = random_kappa(nx, ny, 5, 0.1, 10.0)
    prob = problem(nx, ny, nsx, nsy, K, M=5.0)
    gs = _sim_env(prob, MPM2P_REPAIR="sep")
    gd = _sim_env(prob, MPM2P_REPAIR="dense")
    o = api.Simulator(prob, oracle)
    a, b, r = gs.mrcm_solve(K), gd.mrcm_solve(K), o.mrcm_solve(K)
    for x, y in ((a.p, b.p), (a.u, b.u), (a.p, r.p), (a.u, r.u)):
        assert rel_l2(x, y) <= 1e-10
    kn = K * np.exp(0.05 * np.random.default_rng(7).standard_normal(K.size))
    ma, mr = gs.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
    assert rel_l2(ma.p, mr.p) <= 1e-10 and rel_l2(ma.u, mr.u) <= 1e-10
    sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, eta_mode=api.EPS_RELATIVE, te=25, cfl_safety=0.5)
    ra, rr = gs.run(sp), o.run(sp)
    assert [s["rebuilt"] for s in ra.record.steps] == [s["rebuilt"] for s in rr.record.steps]
    assert np.max(np.abs(ra.s_final - rr.s_final)) <= TOL_S
    assert rel_l2(ra.u_final, rr.u_final) <= TOL_PU


def test_mpm_rhs_per_subdomain_bitwise():
    """k_mpm_rhs_sub (one CTA per subdomain) is bit-identical to one thread per cell."""
    c = configs.build("C2", te_override=31)
    a = _sim_env(c.problem, MPM2P_RHS_W=0, MPM2P_RHS_SUB=1).run(c.split, c.s0())
    b = _sim_env(c.problem, MPM2P_RHS_W=0, MPM2P_RHS_SUB=0).run(c.split, c.s0())
    assert np.array_equal(a.s_final, b.s_final) and np.array_equal(a.u_final, b.u_final)
    assert np.array_equal(a.p_final, b.p_final)


@pytest.mark.parametrize("nx,ny,sx,sy", [(62, 45, 2, 3), (93, 130, 3, 5), (300, 20, 10, 1), (40, 96, 2, 4)])
def test_mpm_rhs_cell_ragged(oracle, nx, ny, sx, sy):
    """k_mpm_rhs_w (one thread per cell, east faces by shuffle inside a
    subdomain, each subdomain's own w on its edges) on ragged grids: the
    MPM-2P update matches the oracle and the per-subdomain kernel."""
    K = random_kappa(nx, ny, 13, 0.1, 10.0)
    for bc in (api.pressure_drop(nx, ny), api.unit_inflow(nx, ny)):
        prob = problem(nx, ny, sx, sy, K, bc=bc)
        a, b, o = _sim_env(prob, MPM2P_RHS_W=1), _sim_env(prob, MPM2P_RHS_W=0), api.Simulator(prob, oracle)
        for sim in (a, b, o):
            sim.mrcm_solve(K)
        kn = K * np.exp(0.1 * np.random.default_rng(2).standard_normal(K.size))
        ma, mb, mo = a.mpm_pressure_update(kn), b.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
        assert rel_l2(ma.u, mo.u) < TOL_PU and rel_l2(ma.p, mo.p) < TOL_PU
        assert rel_l2(ma.u, mb.u) < 1e-12


def test_mpm_edge_cache_across_updates_and_rebuilds(oracle):
    """k_mpm_edges_kn reads the pressure drop and the static g' / rhs terms
    that the rebuild cached (launch_rebuild): several MPM-2P updates with
    different kappa_n after one rebuild, then a second rebuild with another
    kappa_m, with flux faces (z' changes every update), pressure faces and a
    physical Robin side; then a run that alternates MPM-2P updates and
    rebuilds. Everything against the oracle (mpm.cpp:48-86)."""
    from test_robin_faces import robin_slab
    nx, ny = 96, 64
    K = random_kappa(nx, ny, 21, 0.1, 10.0)
    rng = np.random.default_rng(5)
    for bc in (api.unit_inflow(nx, ny), api.pressure_drop(nx, ny), robin_slab(nx, ny, 0.5, 1.0)):
        prob = problem(nx, ny, 3, 2, K, bc=bc)
        g, o = _sim_env(prob, MPM2P_RHS_W=1), api.Simulator(prob, oracle)
        km = K
        for _ in range(2):  # two rebuilds, three updates after each
            g.mrcm_solve(km)
            o.mrcm_solve(km)
            for _ in range(3):
                kn = km * np.exp(0.1 * rng.standard_normal(K.size))
                a, b = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
                assert rel_l2(a.u, b.u) <= 1e-10 and rel_l2(a.p, b.p) <= 1e-10
            km = K * np.exp(0.3 * rng.standard_normal(K.size))
    prob = problem(nx, ny, 3, 2, K, M=5.0, bc=api.unit_inflow(nx, ny))
    sp = api.SplittingConfig(method=api.MPM2P, eta=0.02, eta_mode=api.EPS_RELATIVE, te=60, cfl_safety=0.5)
    ra, rr = _sim_env(prob, MPM2P_RHS_W=1).run(sp), api.Simulator(prob, oracle).run(sp)
    seq = [s["rebuilt"] for s in rr.record.steps]
    assert [s["rebuilt"] for s in ra.record.steps] == seq and 1 < sum(seq) < len(seq)
    assert np.max(np.abs(ra.s_final - rr.s_final)) <= TOL_S
    assert rel_l2(ra.u_final, rr.u_final) <= TOL_PU and rel_l2(ra.p_final, rr.p_final) <= TOL_PU


@pytest.mark.parametrize("nx,nsx", [(64, 4), (96, 4), (64, 2), (128, 4)])
def test_blocked_dmma_downscale_parity(oracle, nx, nsx):
    """The fused downscale on the fp64 tensor cores (band_blk.cuh: 8-pivot
    panels, DMMA Schur updates; B = 16, 24, 32) vs the register-window
    scalar LDL^T and vs the oracle's banded LDL^T (mrcm.cpp:388-427)."""
    K = random_kappa(nx, nx, 4, 1e-2, 1e2)
    prob = problem(nx, nx, nsx, nsx, K, M=5.0)
    gb = _sim_env(prob, MPM2P_DS_BLK=1, MPM2P_DS_SPLIT=0, MPM2P_NO_TWIST=1)
    gr = _sim_env(prob, MPM2P_DS_BLK=0, MPM2P_DS_SPLIT=0, MPM2P_NO_TWIST=1)
    o = api.Simulator(prob, oracle)
    a, b, r = gb.mrcm_solve(K), gr.mrcm_solve(K), o.mrcm_solve(K)
    for x, y in ((a.p, b.p), (a.u, b.u), (a.p, r.p), (a.u, r.u)):
        assert rel_l2(x, y) <= 1e-10
    assert a.info.div_residual <= 1e-10 * a.info.div_scale
    kn = K * np.exp(0.1 * np.random.default_rng(2).standard_normal(K.size))
    ma, mr = gb.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
    assert rel_l2(ma.p, mr.p) <= 1e-10 and rel_l2(ma.u, mr.u) <= 1e-10
    sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, eta_mode=api.EPS_RELATIVE, te=30, cfl_safety=0.5)
    ra, rr = gb.run(sp), o.run(sp)
    assert [s["rebuilt"] for s in ra.record.steps] == [s["rebuilt"] for s in rr.record.steps]
    assert np.max(np.abs(ra.s_final - rr.s_final)) <= TOL_S
    assert rel_l2(ra.u_final, rr.u_final) <= TOL_PU and rel_l2(ra.p_final, rr.p_final) <= TOL_PU



@pytest.mark.parametrize("nx,ny,sx,sy", [(62, 45, 2, 3), (93, 130, 3, 5), (300, 20, 10, 1), (40, 96, 2, 4),
                                         (64, 64, 2, 2)])
def test_velocity_scatter_ragged(oracle, nx, ny, sx, sy):
    """k_ds_u_div on ragged grids (rows that end inside a warp, subdomain
    widths that do not divide 32): east faces by shuffle, the maxima's and
    the CFL's divisions hoisted out of the reductions. MRCM and MPM-2P
    velocities match the oracle to the parity bar, the downscale diagnostics
    to roundoff, and the fused next-step CFL dt of a run equals
    cfl_timestep (transport kernel) of the run's velocity bitwise."""
    K = random_kappa(nx, ny, 3, 0.1, 10.0)
    prob = problem(nx, ny, sx, sy, K)
    g, o = api.Simulator(prob), api.Simulator(prob, oracle)
    sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
    assert rel_l2(sg.u, so.u) < TOL_PU
    assert abs(sg.info.div_scale - so.info.div_scale) <= 1e-12 * so.info.div_scale
    assert sg.info.div_residual <= 1e-10 * sg.info.div_scale
    mg, mo = g.mpm_pressure_update(K * 1.05), o.mpm_pressure_update(K * 1.05)
    assert rel_l2(mg.u, mo.u) < TOL_PU
    sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, te=2, cfl_safety=0.7)
    r = g.run(sp)
    g2 = api.Simulator(prob)
    g2.run_begin(sp)
    s_, p_, u_ = g2.run_read()
    assert r.record.steps[1]["dt"] == g2.cfl_timestep(u_, 0.7, 1.0)
