"""The reference's own known answers, asked of the GPU library directly.

The parity tests compare the CUDA path with the oracle; these restate the
properties the reference's unit tests assert (proj/tests/test_mrcm.cpp,
proj/tests/test_mpm.cpp) and check them on the device through the same entry
points, with the reference's grids, decompositions, boundary data and
tolerances. No oracle is involved: each expected value is analytic, or the
device's own fine solve (solve_cell_centered) where the reference compares
with it. Conductivity fields are seeded random fields (the reference's
sampler is out of scope; the properties hold for any positive field)."""
import numpy as np
import pytest

from cases import problem, random_kappa
from paper_2103_11050_b200 import api

pytestmark = pytest.mark.gpu


def _vfaces(nx, ny, u):
    return u[: ny * (nx + 1)].reshape(ny, nx + 1)


def _hfaces(nx, ny, u):
    return u[ny * (nx + 1):].reshape(ny + 1, nx)


def _flux_err(nx, ny, u, uf, lx=1.0, ly=1.0):
    """Face-area weighted relative L2 flux error (test_mrcm.cpp:633-641)."""
    w = np.concatenate([np.full(ny * (nx + 1), ly / ny), np.full((ny + 1) * nx, lx / nx)])
    return np.sqrt(np.sum(w * (u - uf) ** 2) / np.sum(w * uf ** 2))


def test_zero_data_gives_zero_coefficients():
    """test_mrcm.cpp:395-405."""
    K = random_kappa(8, 8, 2, 0.1, 10.0)
    g = api.Simulator(problem(8, 8, 2, 2, K, bc=api.pressure_drop(8, 8, 0.0, 0.0)))
    g.compute_basis_set(K)
    part, _ = g.solve_particular(g.restrict_physical_data())
    co, cnt = g.solve_interface(part)
    assert cnt.interface_solves == 1 and co.size == 8
    assert np.max(np.abs(co)) <= 1e-12


def test_weak_jump_integrals_vanish_for_random_sources():
    """test_mrcm.cpp:407-426: |flux jump| <= 1e-10 scale, |pressure jump| <= 1e-9 scale."""
    K = random_kappa(8, 8, 2, 0.1, 10.0)
    q = np.random.default_rng(13).uniform(-1.0, 1.0, 64)
    g = api.Simulator(problem(8, 8, 2, 2, K, q=q))
    g.compute_basis_set(K)
    part, _ = g.solve_particular(g.restrict_physical_data())
    co, _ = g.solve_interface(part)
    recon = g.reconstruct(co, part)
    fj, pj = g.weak_continuity_residuals(recon)
    scale = max(float(np.max(np.abs(recon["u"]))), 1.0)  # >= the skeleton traces' size
    assert fj <= 1e-10 * scale and pj <= 1e-9 * scale


def test_uniform_flow_is_reproduced_exactly():
    """test_mrcm.cpp:429-463: K = 1, unit pressure drop: u = 1 on every
    vertical face, 0 on horizontal faces (strip decomposition with constant
    spaces; 2 x 2 with linear spaces)."""
    g = api.Simulator(problem(16, 8, 4, 1, np.ones(128)))
    sol = g.mrcm_solve(np.ones(128))
    assert np.max(np.abs(_vfaces(16, 8, sol.u) - 1.0)) <= 1e-8
    g = api.Simulator(problem(8, 8, 2, 2, np.ones(64), space=api.SPACE_LINEAR))
    sol = g.mrcm_solve(np.ones(64))
    assert np.max(np.abs(_vfaces(8, 8, sol.u) - 1.0)) <= 1e-8
    assert np.max(np.abs(_hfaces(8, 8, sol.u))) <= 1e-8


def test_reconstruction_linearity():
    """test_mrcm.cpp:465-507: doubling q and the boundary values doubles the
    reconstructed pressure (same basis set); zero coefficients reproduce the
    particular solution exactly."""
    K = random_kappa(8, 8, 31, 0.1, 10.0)
    q = np.random.default_rng(17).uniform(-1.0, 1.0, 64)
    g = api.Simulator(problem(8, 8, 2, 2, K, q=q))
    g.compute_basis_set(K)
    d1 = g.restrict_physical_data()
    p1, _ = g.solve_particular(d1)
    c1, _ = g.solve_interface(p1)
    r1 = g.reconstruct(c1, p1)
    d2 = dict(d1, q=2.0 * d1["q"], value=2.0 * d1["value"])
    p2, _ = g.solve_particular(d2)
    c2, _ = g.solve_interface(p2)
    r2 = g.reconstruct(c2, p2)
    assert np.max(np.abs(r2["p"] - 2.0 * r1["p"])) <= 1e-10
    rz = g.reconstruct(np.zeros_like(c1), p1)
    assert np.array_equal(rz["p"], p1["p"])


def test_mrcm_equals_the_fine_solver_in_the_equivalent_limits():
    """test_mrcm.cpp:576-612: a 1 x 1 decomposition is the fine solve (1e-10);
    per-edge constant spaces reproduce the undecomposed solution (1e-8 of max|u|)."""
    K = random_kappa(12, 10, 51, 1e-2, 1e2)
    q = np.zeros(120)
    q[3 * 12 + 2] = 5.0
    g = api.Simulator(problem(12, 10, 1, 1, K, q=q))
    sol, (pf, uf) = g.mrcm_solve(K), g.fine_solve(K)
    assert np.max(np.abs(sol.u - uf)) <= 1e-10 and np.max(np.abs(sol.p - pf)) <= 1e-10
    K = random_kappa(16, 16, 52, 0.1, 10.0)
    g = api.Simulator(problem(16, 16, 2, 2, K, hbar=api.HBAR_PER_EDGE))
    sol, (pf, uf) = g.mrcm_solve(K), g.fine_solve(K)
    assert np.max(np.abs(sol.u - uf)) <= 1e-8 * np.max(np.abs(uf))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_richness_monotonicity_of_the_flux_error(seed):
    """test_mrcm.cpp:614-650: e(H/2) <= 1.05 e(H), e(h) <= 1.05 e(H/2), and
    the per-edge space is exact (<= 1e-7)."""
    K = random_kappa(32, 32, seed, 0.05, 20.0)
    errs = []
    for hbar in (api.HBAR_WHOLE, api.HBAR_HALF, api.HBAR_PER_EDGE):
        g = api.Simulator(problem(32, 32, 4, 4, K, hbar=hbar))
        sol, (_, uf) = g.mrcm_solve(K), g.fine_solve(K)
        errs.append(_flux_err(32, 32, sol.u, uf))
    eH, eH2, eh = errs
    assert eH2 <= 1.05 * eH and eh <= 1.05 * eH2 and eh <= 1e-7


@pytest.mark.parametrize("nsx,bc", [(4, "pd"), (2, "ui")])
def test_zero_perturbation_idempotence(nsx, bc):
    """test_mpm.cpp:94-137: an MPM-2P update with kappa_n = kappa_m returns
    the MRCM solution (1e-8 of max|u|); under flux-driven boundaries the
    imposed inflow is reproduced exactly (1e-9)."""
    K = random_kappa(16, 16, 4 if bc == "pd" else 8, 0.1, 10.0)
    spec = api.pressure_drop(16, 16) if bc == "pd" else api.unit_inflow(16, 16)
    g = api.Simulator(problem(16, 16, nsx, nsx, K, bc=spec))
    sol = g.mrcm_solve(K)
    r = g.mpm_pressure_update(K)
    assert np.max(np.abs(r.u - sol.u)) <= 1e-8 * np.max(np.abs(sol.u))
    assert np.max(np.abs(r.p - sol.p)) <= 1e-8
    if bc == "ui":
        assert np.max(np.abs(_vfaces(16, 16, r.u)[:, 0] - 1.0)) <= 1e-9


def test_uniform_conductivity_doubling_is_recovered_exactly():
    """test_mpm.cpp:139-154: kappa 1 -> 2 doubles u and keeps p (1e-9)."""
    g = api.Simulator(problem(16, 16, 4, 4, np.ones(256)))
    sol = g.mrcm_solve(np.ones(256))
    r = g.mpm_pressure_update(np.full(256, 2.0))
    assert np.max(np.abs(r.u - 2.0 * sol.u)) <= 1e-9 and np.max(np.abs(r.p - sol.p)) <= 1e-9


def test_an_mpm_step_is_n_particular_and_n_downscale_solves():
    """test_mpm.cpp:156-175 and the rebuild ledger of test_mrcm.cpp:269-307:
    96 homogeneous + 16 particular + 16 downscale solves and one interface
    solve for a 4 x 4 rebuild; 0 / 16 / 16 / 1 for the MPM-2P update."""
    K = random_kappa(16, 16, 11, 0.1, 10.0)
    g = api.Simulator(problem(16, 16, 4, 4, K))
    c = g.mrcm_solve(K).counters
    assert (c.homogeneous, c.particular, c.downscale, c.interface_solves) == (96, 16, 16, 1)
    c2 = g.mpm_pressure_update(1.003 * K).counters
    assert (c2.homogeneous, c2.particular, c2.downscale, c2.interface_solves) == (0, 16, 16, 1)


def test_mpm_reuses_the_stored_interface_matrix_bytes():
    """test_mpm.cpp:177-197."""
    K = np.random.default_rng(3).uniform(0.5, 2.0, 64)
    g = api.Simulator(problem(8, 8, 2, 2, K))
    g.mrcm_solve(K)
    M0 = g.interface_matrix().copy()
    g.mpm_pressure_update(1.004 * K)
    assert M0.tobytes() == g.interface_matrix().tobytes()


def test_mpm_velocity_is_conservative_under_the_new_conductivity():
    """test_mpm.cpp:199-222: |div u - q| <= 1e-10 max_f |u_f| area_f / vol."""
    nx = ny = 16
    K = random_kappa(nx, ny, 23, 0.1, 10.0)
    g = api.Simulator(problem(nx, ny, 4, 4, K))
    g.mrcm_solve(K)
    r = g.mpm_pressure_update(K * np.random.default_rng(99).uniform(1.0, 1.02, K.size))
    scale = np.max(np.abs(r.u)) * (1.0 / nx) / (1.0 / (nx * ny))
    assert np.max(np.abs(g.divergence(r.u))) <= 1e-10 * scale


def test_mpm_accuracy_stays_comparable_to_a_fresh_mrcm_solve():
    """test_mpm.cpp:224-259: after a smooth 1 % drift the reused-basis flux
    error is within a factor two of a fresh multiscale solve's."""
    nx = ny = 32
    K = random_kappa(nx, ny, 31, 0.1, 10.0)
    xc, yc = (np.arange(nx) + 0.5) / nx, (np.arange(ny) + 0.5) / ny
    K2 = K * (1.0 + 0.01 * np.outer(np.cos(2.0 * yc), np.sin(3.0 * xc)).ravel())
    g = api.Simulator(problem(nx, ny, 4, 4, K))
    g.mrcm_solve(K)
    mpm = g.mpm_pressure_update(K2)
    fresh = g.mrcm_solve(K2)  # compute_beta(kappa2) inside
    _, uf = g.fine_solve(K2)
    assert _flux_err(nx, ny, mpm.u, uf) <= 2.0 * _flux_err(nx, ny, fresh.u, uf) + 1e-12


# ---- transport (proj/tests/test_transport.cpp) ----

def test_mobility_values():
    """test_transport.cpp:13-25 through conductivity = K lambda(S) with K = 1:
    lambda(0) = 1, lambda(1) = M, lambda(0.5) = 10.25 at M = 40; saturations
    outside [0, 1] are clamped (:39-46)."""
    g = api.Simulator(problem(4, 1, 1, 1, np.ones(4), M=40.0))
    lam = g.conductivity(np.array([0.0, 1.0, 0.5, -0.1]))
    assert lam[0] == 1.0 and lam[1] == 40.0 and lam[3] == 1.0
    assert abs(lam[2] - 10.25) <= 1e-15 * 10.25


def test_cfl_time_step():
    """test_transport.cpp:48-71: uniform unit flow at M = 1 gives
    dt = 0.9 h / max f', max f' = 2; doubling u halves dt; zero u returns the cap."""
    nx = ny = 64  # the transport calls do not see the decomposition (2 x 2: the subdomain width limit is 32)
    g = api.Simulator(problem(nx, ny, 2, 2, np.ones(nx * ny), M=1.0))
    u = np.zeros(g.faces)
    u[: ny * (nx + 1)] = 1.0
    assert abs(g.max_fractional_flow_slope() - 2.0) <= 2e-4
    dt = g.cfl_timestep(u, 0.9, 1.0)
    assert abs(dt - 0.9 / 64 / 2.0) <= 1e-3 * dt
    assert abs(g.cfl_timestep(2.0 * u, 0.9, 1.0) - dt / 2.0) <= 1e-12 * dt
    assert g.cfl_timestep(np.zeros(g.faces), 0.9, 1.0) == 1.0


def test_upwind_step_basics():
    """test_transport.cpp:73-99: a divergence-free uniform flow keeps a
    constant state (1e-14), zero velocity leaves s unchanged bit for bit, a
    CFL violation is a NumericError."""
    nx = ny = 16
    g = api.Simulator(problem(nx, ny, 1, 1, np.ones(nx * ny), M=2.0))
    u = np.zeros(g.faces)
    u[: ny * (nx + 1)] = 1.0
    s2 = g.upwind_step(np.full(nx * ny, 0.3), 0.3, u, 1e-3)
    assert np.max(np.abs(s2 - 0.3)) <= 1e-14 * 0.3
    s = np.zeros(nx * ny)
    s[4 * nx + 4] = 0.7
    assert np.array_equal(g.upwind_step(s, 1.0, np.zeros(g.faces), 1e-2), s)
    g1 = api.Simulator(problem(nx, ny, 1, 1, np.ones(nx * ny), M=1.0))
    with pytest.raises(api.NumericError):
        g1.upwind_step(np.zeros(nx * ny), 1.0, u, 1.0)


def test_maximum_principle_and_mass_balance_over_random_steps():
    """test_transport.cpp:143-200: velocities from divergence-free elliptic
    solves (the device's fine solve), random saturations between bursts of
    upwind steps; per step the water volume changes by the boundary fluxes
    times dt (1e-12) and s stays inside [min(s, inflow), max(s, inflow)]."""
    nx = ny = 16
    M, vol, hy = 5.0, 1.0 / (nx * ny), 1.0 / ny
    rng = np.random.default_rng(77)

    def f(sv):
        sv = np.clip(sv, 0.0, 1.0)
        return M * sv * sv / (M * sv * sv + (1.0 - sv) ** 2)

    steps = 0
    while steps < 1500:
        K = np.exp(rng.uniform(-1.5, 1.5, nx * ny))
        bc = api.BoundarySpec.uniform(nx, ny, (api.PRESSURE, 1.0 + rng.uniform()), (api.PRESSURE, 0.0),
                                      (api.FLUX, 0.0), (api.FLUX, 0.0))
        g = api.Simulator(problem(nx, ny, 1, 1, K, bc=bc, M=M))
        _, u = g.fine_solve(K)
        inflow = rng.uniform()
        s = rng.uniform(0.0, 1.0, nx * ny)
        lo, hi = min(s.min(), inflow), max(s.max(), inflow)
        dt = g.cfl_timestep(u, 0.9, 1.0)
        uw, ue = u[: ny * (nx + 1)].reshape(ny, nx + 1)[:, 0], u[: ny * (nx + 1)].reshape(ny, nx + 1)[:, nx]
        for _ in range(100):
            sg = s.reshape(ny, nx)
            b_in = np.where(uw > 0, f(inflow) * uw * hy, -f(sg[:, 0]) * (-uw) * hy).sum()
            b_in += np.where(ue > 0, -f(sg[:, nx - 1]) * ue * hy, f(inflow) * (-ue) * hy).sum()
            s2 = g.upwind_step(s, inflow, u, dt)
            steps += 1
            assert abs((s2.sum() - s.sum()) * vol - b_in * dt) <= 1e-12
            assert s2.min() >= lo - 1e-12 and s2.max() <= hi + 1e-12
            s = s2
        g.close()


# ---- driver accounting (proj/tests/test_simulation.cpp) ----

def _small(method, eta=0.01, te=3):
    """small_inputs (test_simulation.cpp:14-24): the gaussian-slab-small preset's
    shape (config.cpp:433-442: 8 x 8 cells, 2 x 2 subdomains, M = 40, pressure
    drop) on a seeded random field, with the reference's default track_errors =
    true (simulation.hpp:31): a fine reference advances in lockstep and sets
    the transport-step schedule."""
    K = random_kappa(8, 8, 2, 0.2, 5.0)
    prob = problem(8, 8, 2, 2, K, M=40.0)
    return prob, api.SplittingConfig(method=method, eta=eta, te=te, stop_on_breakthrough=False, track_errors=True)


def test_mrcm_every_step_baseline_accounting():
    """test_simulation.cpp:66-79."""
    prob, sp = _small(api.MRCM_EVERY_STEP)
    r = api.Simulator(prob).run(sp).record
    assert r.te == 3 and r.tm_total == 3 and len(r.steps) == 3 and all(s["rebuilt"] == 1 for s in r.steps)
    assert r.nhat == 16
    assert (r.counters.homogeneous, r.counters.particular, r.counters.downscale) == (48, 12, 12)


def test_static_flow_one_rebuild_all_later_steps_reuse():
    """test_simulation.cpp:81-95: no injection, so kappa never changes and epsilon stays zero."""
    prob, sp = _small(api.MPM2P, 0.01, 4)
    r = api.Simulator(prob).run(sp, np.zeros(64), 0.0).record
    assert r.te == 4 and r.tm_total == 1 and r.tm_updates == 0
    assert all(s["epsilon"] == 0.0 for s in r.steps)
    assert (r.counters.homogeneous, r.counters.particular, r.counters.downscale) == (16, 16, 16)


def test_no_updates_never_rebuilds_and_runs_share_the_schedule():
    """test_simulation.cpp:131-148: mpm2p-no-updates rebuilds at step 0 only;
    the three methods share dt and PVI bit for bit."""
    runs = []
    for m in (api.MPM2P, api.MRCM_EVERY_STEP, api.MPM2P_NO_UPDATES):
        prob, sp = _small(m, 0.01, 5)
        runs.append(api.Simulator(prob).run(sp).record)
    a, b, c = runs
    assert c.tm_total == 1 and c.update_steps == [0]
    assert [s["dt"] for s in a.steps] == [s["dt"] for s in b.steps] == [s["dt"] for s in c.steps]
    assert [s["pvi"] for s in a.steps] == [s["pvi"] for s in b.steps]


def test_solve_counters_reconcile_with_the_cost_formulas():
    """test_simulation.cpp:150-157."""
    prob, sp = _small(api.MPM2P, 0.01, 6)
    r = api.Simulator(prob).run(sp).record
    assert r.counters.homogeneous == r.nhat * r.tm_total
    assert r.counters.particular == r.n_sub * r.te and r.counters.downscale == r.n_sub * r.te
    assert r.counters.interface_solves == r.te


def test_velocities_delivered_to_transport_are_conservative():
    """test_simulation.cpp:159-168."""
    prob, sp = _small(api.MPM2P, 0.01, 5)
    g = api.Simulator(prob)
    res = g.run(sp)
    assert res.record.max_div_residual <= 1e-8
    scale = np.max(np.abs(res.u_final)) * (1.0 / 8) / (1.0 / 64)
    assert np.max(np.abs(g.divergence(res.u_final))) <= 1e-10 * scale


def test_fine_reference_runs_record_zero_errors():
    """test_simulation.cpp:123-129."""
    prob, sp = _small(api.FINE_REFERENCE, 0.01, 3)
    r = api.Simulator(prob).run(sp).record
    assert all(s["flux_err"] == 0.0 and s["sat_err"] == 0.0 for s in r.steps)
    assert r.counters.homogeneous == 0


# ---- the fine solve, solve_cell_centered (proj/tests/test_elliptic.cpp) ----

def test_fine_conservation_on_rough_fields():
    """test_elliptic.cpp:89-97: a source / sink pair on a 1e-3 .. 1e3 field,
    conservation_residual <= 1e-10 residual_scale."""
    K = random_kappa(20, 20, 3, 1e-3, 1e3)
    q = np.zeros(400)
    q[4 * 20 + 3], q[12 * 20 + 15] = 400.0, -400.0
    g = api.Simulator(problem(20, 20, 1, 1, K, q=q))
    g.fine_solve(K)
    _, _, res, scale = g.fine_stats()
    assert res <= 1e-10 * scale


def test_fine_mirror_symmetry():
    """test_elliptic.cpp:99-118: with kappa symmetric about x = lx/2, swapping
    the left and right pressures mirrors p and reverses the flux."""
    nx, ny = 10, 6
    K = random_kappa(nx, ny, 11).reshape(ny, nx)
    K[:, nx // 2:] = K[:, : nx // 2][:, ::-1]
    K = K.ravel()
    a = api.Simulator(problem(nx, ny, 1, 1, K, bc=api.pressure_drop(nx, ny, 1.0, 0.0)))
    b = api.Simulator(problem(nx, ny, 1, 1, K, bc=api.pressure_drop(nx, ny, 0.0, 1.0)))
    (pa, ua), (pb, ub) = a.fine_solve(K), b.fine_solve(K)
    assert np.max(np.abs(pb.reshape(ny, nx) - pa.reshape(ny, nx)[:, ::-1])) <= 1e-11
    assert np.max(np.abs(_vfaces(nx, ny, ub) + _vfaces(nx, ny, ua)[:, ::-1])) <= 1e-10 * np.max(np.abs(ua))


def test_fine_scaling_kappa_scales_u_and_leaves_p():
    """test_elliptic.cpp:120-132 (10 x 8 cells instead of 9 x 7: the device
    fine solve's block preconditioner has kernels for widths 4, 8, 10, 12, 16,
    20, 24, 32)."""
    K = random_kappa(10, 8, 5)
    g = api.Simulator(problem(10, 8, 1, 1, K))
    (pa, ua), (pb, ub) = g.fine_solve(K), g.fine_solve(3.0 * K)
    assert np.max(np.abs(pb - pa)) <= 1e-11 and np.max(np.abs(ub - 3.0 * ua)) <= 1e-11
