"""Pins the CPU oracle (the parity checker) against the reference's own
recorded results and known answers. No GPU needed.

Golden: tests/golden/reference_recorded.json = proj/test_output.txt:7-22.
Known answers follow proj/tests/test_{elliptic,transport,mpm,mrcm,simulation}.cpp.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from cases import problem, random_kappa
from paper_2103_11050_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_recorded.json")))


def osim(prob, oracle):
    return api.Simulator(prob, oracle)


def test_slab_study_reproduces_recorded_reference_run():
    """acceptance.cpp:122-164 run_slab_study(303) vs proj/test_output.txt:7-22."""
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "pin_slab"], check=True)
    out = subprocess.run([os.path.join(odir, "pin_slab"), "303"], check=True, capture_output=True, text=True).stdout
    r = json.loads(out)
    assert r["te"] == GOLD["te"]
    assert abs(r["bt_pvi"] - GOLD["bt_pvi"]) < 1e-6
    for k, v in GOLD["rebuilds"].items():
        assert r["rebuilds"][k] == v, k
    for k, v in GOLD["flux_err"].items():
        assert abs(r["flux_err"][k] - v) <= 5e-5 * abs(v) + 1e-6, (k, r["flux_err"][k], v)
    for k, v in GOLD["sat_err"].items():
        assert abs(r["sat_err"][k] - v) <= 5e-5 * abs(v) + 1e-6, (k, r["sat_err"][k], v)
    assert r["nhat"] == GOLD["nhat"]
    assert abs(r["rcr"] - GOLD["rcr_from_run"]) < 1e-3
    assert r["max_div_ratio"] <= GOLD["max_div_ratio_bound"]


def test_rcr_worked_examples():
    for nhat, n, te, tm, want in GOLD["rcr_examples"]:
        assert abs(api.rcr(nhat, n, te, tm) - want) <= 0.01
    assert api.rcr(96, 16, 3500, 3500) == 0.0
    with pytest.raises(api.ConfigError):
        api.rcr(96, 16, 0, 0)


def test_linear_pressure_unit_flux(oracle):
    """test_elliptic.cpp:59-73 (fine solve, kappa = 1, pressure drop)."""
    import ctypes as C
    nx, ny = 16, 8
    s = osim(problem(nx, ny, 1, 1, np.ones(nx * ny)), oracle)
    p, u = np.empty(nx * ny), np.empty(s.faces)
    K = np.ones(nx * ny)
    assert oracle.dll.oracle_fine_solve(s.h, api.dptr(K), api.dptr(p), api.dptr(u)) == 0
    x = (np.arange(nx) + 0.5) / nx
    np.testing.assert_allclose(p.reshape(ny, nx), np.broadcast_to(1.0 - x, (ny, nx)), atol=1e-12)
    nv = (nx + 1) * ny
    np.testing.assert_allclose(u[:nv], 1.0, atol=1e-12)
    np.testing.assert_allclose(u[nv:], 0.0, atol=1e-12)
    del C


def test_layered_flux_proportional_to_kappa(oracle):
    """test_elliptic.cpp:75-87."""
    nx = ny = 8
    K = np.where(np.arange(ny)[:, None] < ny // 2, 1.0, 4.0) * np.ones((ny, nx))
    s = osim(problem(nx, ny, 1, 1, K.ravel()), oracle)
    p, u = np.empty(nx * ny), np.empty(s.faces)
    assert oracle.dll.oracle_fine_solve(s.h, api.dptr(K.ravel()), api.dptr(p), api.dptr(u)) == 0
    uv = u[:(nx + 1) * ny].reshape(ny, nx + 1)
    want = np.where(np.arange(ny)[:, None] < ny // 2, 1.0, 4.0)
    np.testing.assert_allclose(uv, np.broadcast_to(want, uv.shape), rtol=1e-11)


def test_epsilon_closed_forms(oracle):
    """test_mpm.cpp:50-71."""
    nx = ny = 64
    s = osim(problem(nx, ny, 1, 1, np.ones(nx * ny)), oracle)
    a = np.ones(nx * ny)
    assert s.epsilon(a, a, api.EPS_RELATIVE) == 0.0
    assert abs(s.epsilon(a * 1.01, a, api.EPS_RELATIVE) - 0.01) < 1e-12
    b = a.copy()
    b[20 * nx + 10] = 2.0
    assert abs(s.epsilon(b, a, api.EPS_RELATIVE) - 1.0 / 64) < 1e-14
    assert abs(s.epsilon(b, a, api.EPS_ABSOLUTE) - 1.0 / 64) < 1e-14
    with pytest.raises(api.ConfigError):
        s.epsilon(b, a, api.EPS_MOBILITY)


def test_mobility_fractional_flow_values(oracle):
    """test_transport.cpp:13-25 through conductivity (K=1) and injection_rate."""
    nx, ny = 10, 10
    s = osim(problem(nx, ny, 1, 1, np.ones(nx * ny), M=40.0), oracle)
    sat = np.zeros(nx * ny)
    sat[:3] = [0.0, 1.0, 0.5]
    k = s.conductivity(sat)
    assert k[0] == 1.0 and k[1] == 40.0 and abs(k[2] - 10.25) < 1e-15
    u = np.zeros(s.faces)
    for j in range(ny):
        u[j * (nx + 1)] = 1.0  # inflow through the west side
        u[j * (nx + 1) + nx] = 1.0
    # injected water rate = f(s_bar) * u * ly (simulation.cpp:85-101)
    assert abs(s.injection_rate(u, 0.5) - 40.0 / 41.0) < 1e-14
    assert abs(s.injection_rate(u, 1.0) - 1.0) < 1e-14


def test_cfl_uniform_flow(oracle):
    """test_transport.cpp:48-71."""
    nx = ny = 64
    s = osim(problem(nx, ny, 1, 1, np.ones(nx * ny), M=1.0), oracle)
    assert abs(s.max_fractional_flow_slope() - 2.0) < 2e-4
    u = np.zeros(s.faces)
    u[:(nx + 1) * ny] = 1.0
    dt = s.cfl_timestep(u, 0.9, 1.0)
    assert abs(dt - 0.9 * (1.0 / 64) / 2.0) < 1e-3 * dt
    assert abs(s.cfl_timestep(2 * u, 0.9, 1.0) - dt / 2) < 1e-12
    assert s.cfl_timestep(np.zeros(s.faces), 0.9, 1.0) == 1.0


def test_upwind_front_matches_independent_1d(oracle):
    """test_transport.cpp:101-141."""
    n = 200
    s = osim(problem(n, 1, 1, 1, np.ones(n), lx=1.0, ly=1.0 / n, M=1.0), oracle)
    u = np.zeros(s.faces)
    u[:n + 1] = 1.0
    dt = s.cfl_timestep(u, 0.9, 1.0)
    sat = np.zeros(n)
    for _ in range(150):
        sat = s.upwind_step(sat, 1.0, u, dt)
    r = np.zeros(n)
    h = 1.0 / n
    f = lambda v: v * v / (v * v + (1 - v) * (1 - v))  # noqa: E731
    for _ in range(150):
        flux = f(np.concatenate([[1.0], r]))
        r = r - dt / h * (flux[1:] - flux[:-1])
    front = lambda a: int(np.max(np.nonzero(a > 0.5)[0])) if np.any(a > 0.5) else 0  # noqa: E731
    assert abs(front(sat) - front(r)) <= 1 and front(r) > 5


def test_upwind_mass_balance_and_max_principle(oracle):
    """test_transport.cpp:143-200 (shortened: 600 steps)."""
    nx = ny = 16
    rng = np.random.default_rng(77)
    M = 5.0
    steps = 0
    while steps < 600:
        K = np.exp(rng.uniform(-1.5, 1.5, nx * ny))
        bc = api.pressure_drop(nx, ny, 1.0 + rng.uniform(), 0.0)
        s = osim(problem(nx, ny, 1, 1, K, bc=bc, M=M), oracle)
        p, u = np.empty(nx * ny), np.empty(s.faces)
        assert oracle.dll.oracle_fine_solve(s.h, api.dptr(K), api.dptr(p), api.dptr(u)) == 0
        inflow = rng.uniform()
        sat = rng.uniform(0, 1, nx * ny)
        lo, hi = min(sat.min(), inflow), max(sat.max(), inflow)
        dt = s.cfl_timestep(u, 0.9, 1.0)
        f = lambda v: M * v * v / (M * v * v + (1 - v) ** 2)  # noqa: E731
        for _ in range(100):
            m0 = sat.sum() / (nx * ny)
            uw = u[np.arange(ny) * (nx + 1)]
            ue = u[np.arange(ny) * (nx + 1) + nx]
            s_w, s_e = sat.reshape(ny, nx)[:, 0], sat.reshape(ny, nx)[:, -1]
            net_in = (np.where(uw > 0, f(inflow) * uw, f(s_w) * uw).sum()
                      - np.where(ue > 0, f(s_e) * ue, f(inflow) * ue).sum()) / ny
            sat = s.upwind_step(sat, inflow, u, dt)
            m1 = sat.sum() / (nx * ny)
            assert abs(m1 - m0 - net_in * dt) <= 1e-12 * max(1.0, abs(m0))
            assert sat.min() >= lo - 1e-12 and sat.max() <= hi + 1e-12
            steps += 1


def _monolithic(nx, ny, nsx, nsy, K, q, bc, space_kind, hbar, beta, lx=1.0, ly=1.0):
    """Independent oracle: the whole Robin-coupled system as one dense matrix
    (proj/tests/test_mrcm.cpp:39-170), built here from the geometry in numpy."""
    hx, hy = lx / nx, ly / ny
    snx, sny = nx // nsx, ny // nsy
    ns = nsx * nsy
    NV, NH = nsy * (nsx - 1), (nsy - 1) * nsx

    def iface_edges(k):
        return sny if k < NV else snx

    # bases per interface (interface_space.cpp:9-52)
    bases = []
    for k in range(NV + NH):
        n = iface_edges(k)
        if space_kind == api.SPACE_LINEAR:
            bases.append([np.ones(n), 2.0 * (np.arange(n) + 0.5) / n - 1.0])
        else:
            seg = {api.HBAR_WHOLE: n, api.HBAR_HALF: n // 2, api.HBAR_PER_EDGE: 1}[hbar]
            bases.append([np.where((np.arange(n) >= t) & (np.arange(n) < t + seg), 1.0, 0.0)
                          for t in range(0, n, seg)])
    first, nb = [], 0
    for b in bases:
        first.append(nb)
        nb += len(b)
    nu = npres = nb
    ncell = nx * ny
    u_off, p_off = ncell, ncell + nu
    dim = ncell + nu + npres
    A = np.zeros((dim, dim))
    rhs = np.zeros(dim)
    Kg = K.reshape(ny, nx)
    qg = q.reshape(ny, nx)
    vol = hx * hy
    harm = lambda a, b: 2 * a * b / (a + b)  # noqa: E731
    bidx = {}
    off = 0
    for k in range(NV + NH):
        bidx[k] = off
        off += iface_edges(k)
    for s in range(ns):
        sx, sy = s % nsx, s // nsx
        i0, j0 = sx * snx, sy * sny
        row = lambda ii, jj: (j0 + jj) * nx + (i0 + ii)  # noqa: E731
        for jj in range(sny):
            for ii in range(snx):
                r = row(ii, jj)
                rhs[r] += qg[j0 + jj, i0 + ii] * vol
                for di, dj, area, dist in ((-1, 0, hy, hx), (1, 0, hy, hx), (0, -1, hx, hy), (0, 1, hx, hy)):
                    a, b = ii + di, jj + dj
                    if 0 <= a < snx and 0 <= b < sny:
                        t = harm(Kg[j0 + jj, i0 + ii], Kg[j0 + b, i0 + a]) * area / dist
                        A[r, r] += t
                        A[r, row(a, b)] -= t
        # boundary edges W,E,S,N
        edges = []
        for jj in range(sny):
            edges.append(("W", 0, jj, -1.0, (sx > 0), sy * (nsx - 1) + sx - 1, jj, j0 + jj))
        for jj in range(sny):
            edges.append(("E", snx - 1, jj, 1.0, (sx < nsx - 1), sy * (nsx - 1) + sx, jj, ny + j0 + jj))
        for ii in range(snx):
            edges.append(("S", ii, 0, -1.0, (sy > 0), NV + (sy - 1) * nsx + sx, ii, 2 * ny + i0 + ii))
        for ii in range(snx):
            edges.append(("N", ii, sny - 1, 1.0, (sy < nsy - 1), NV + sy * nsx + sx, ii, 2 * ny + nx + i0 + ii))
        for side, ii, jj, sign, skel, k, pos, g in edges:
            area = hy if side in "WE" else hx
            th = Kg[j0 + jj, i0 + ii] * area / ((hx if side in "WE" else hy) / 2.0)
            r = row(ii, jj)
            if skel:
                bt = beta[0][bidx[k] + pos] if sign > 0 else beta[1][bidx[k] + pos]
                te = 1.0 / (1.0 / th + bt / area)
                A[r, r] += te
                for t, phi in enumerate(bases[k]):
                    A[r, u_off + first[k] + t] += te * bt * sign * phi[pos]
                    A[r, p_off + first[k] + t] -= te * phi[pos]
                # weak rows
                def add_unout(wrow, w):
                    A[wrow, r] += w * te / area
                    for t, phi in enumerate(bases[k]):
                        A[wrow, u_off + first[k] + t] += w * te * bt * sign * phi[pos] / area
                        A[wrow, p_off + first[k] + t] -= w * te * phi[pos] / area
                for t, psi in enumerate(bases[k]):
                    add_unout(u_off + first[k] + t, psi[pos] * area)
                for t, phr in enumerate(bases[k]):
                    wr = u_off + npres + first[k] + t
                    add_unout(wr, bt * phr[pos] * sign * area)
                    for t2, phb in enumerate(bases[k]):
                        A[wr, u_off + first[k] + t2] -= bt * phb[pos] * sign * phr[pos] * sign * area
            else:
                if bc.kind[g] == api.PRESSURE:
                    A[r, r] += th
                    rhs[r] += th * bc.value[g]
                else:
                    rhs[r] -= bc.value[g] * area
    x = np.linalg.solve(A, rhs)
    return x[u_off:u_off + nu], x[p_off:p_off + npres]


@pytest.mark.parametrize("nx,ny,nsx,nsy,space,hbar,bcname,alpha", [
    (8, 8, 2, 2, api.SPACE_CONSTANT, api.HBAR_WHOLE, "pd", api.ALPHA_UNIFORM),
    (8, 8, 2, 2, api.SPACE_CONSTANT, api.HBAR_HALF, "pd", api.ALPHA_UNIFORM),
    (8, 8, 2, 2, api.SPACE_LINEAR, api.HBAR_WHOLE, "pd", api.ALPHA_UNIFORM),
    (12, 6, 3, 2, api.SPACE_LINEAR, api.HBAR_WHOLE, "ui", api.ALPHA_ADAPTIVE),
])
def test_oracle_matches_monolithic_system(oracle, nx, ny, nsx, nsy, space, hbar, bcname, alpha):
    """test_mrcm.cpp:309-385: U, P coefficients match the monolithic dense solve to 1e-8."""
    lx = 2.0 if nx == 12 else 1.0
    K = random_kappa(nx, ny, 21, 1e-2 if alpha else 0.3, 1e2 if alpha else 3.0)
    q = np.random.default_rng(5).uniform(-1, 1, nx * ny)
    bc = api.pressure_drop(nx, ny) if bcname == "pd" else api.unit_inflow(nx, ny)
    prob = problem(nx, ny, nsx, nsy, K, bc=bc, lx=lx, q=q, space=space, hbar=hbar,
                   alpha=api.AlphaSpec(mode=alpha))
    s = osim(prob, oracle)
    beta = s.compute_beta(K)
    sol = s.mrcm_solve(K)
    U, P = _monolithic(nx, ny, nsx, nsy, K, q, bc, space, hbar, beta, lx=lx)
    scale = max(1.0, np.abs(sol.p).max())
    np.testing.assert_allclose(sol.coeffs[:len(U)], U, atol=1e-8 * scale, rtol=1e-8)
    np.testing.assert_allclose(sol.coeffs[len(U):], P, atol=1e-8 * scale, rtol=1e-8)


def test_basis_counts_and_mpm_ledger(oracle):
    """test_mrcm.cpp:269-307, test_mpm.cpp:156-175."""
    nx = ny = 16
    K = random_kappa(nx, ny, 1)
    s = osim(problem(nx, ny, 4, 4, K), oracle)
    sol = s.mrcm_solve(K)
    assert (sol.counters.homogeneous, sol.counters.particular, sol.counters.downscale) == (96, 16, 16)
    assert s.dim == 48
    m = s.mpm_pressure_update(K * 1.003)
    c = m.counters
    assert (c.homogeneous, c.particular, c.downscale, c.interface_solves) == (0, 16, 16, 1)


def test_zero_perturbation_idempotence(oracle):
    """test_mpm.cpp:94-137: MPM with kappa_n = kappa_m reproduces the MRCM solution."""
    nx = ny = 16
    K = random_kappa(nx, ny, 4, 0.1, 10.0)
    s = osim(problem(nx, ny, 4, 4, K), oracle)
    sol = s.mrcm_solve(K)
    m = s.mpm_pressure_update(K)
    umax = np.abs(sol.u).max()
    np.testing.assert_allclose(m.u, sol.u, atol=1e-8 * umax)
    np.testing.assert_allclose(m.p, sol.p, atol=1e-8)


def test_driver_semantics(oracle):
    """test_simulation.cpp:66-157: every-step accounting, eta=0 equivalence,
    static flow, ledger reconciliation."""
    nx = ny = 8
    K = random_kappa(nx, ny, 2, 0.5, 2.0)
    prob = problem(nx, ny, 2, 2, K, M=40.0)
    s = osim(prob, oracle)
    every = s.run(api.SplittingConfig(method=api.MRCM_EVERY_STEP, te=3))
    assert every.record.te == 3 and every.record.tm_total == 3 and every.record.nhat == 16
    assert every.record.counters.homogeneous == 48 and every.record.counters.downscale == 12
    a = s.run(api.SplittingConfig(method=api.MPM2P, eta=0.0, te=4))
    b = s.run(api.SplittingConfig(method=api.MRCM_EVERY_STEP, te=4))
    assert [x["rebuilt"] for x in a.record.steps] == [x["rebuilt"] for x in b.record.steps]
    assert np.array_equal(a.s_final, b.s_final)
    static = s.run(api.SplittingConfig(method=api.MPM2P, eta=0.01, te=4), inflow_sat=0.0)
    assert static.record.tm_total == 1 and all(x["epsilon"] == 0.0 for x in static.record.steps)
    r = s.run(api.SplittingConfig(method=api.MPM2P, eta=0.01, te=6)).record
    assert r.counters.homogeneous == r.nhat * r.tm_total
    assert r.counters.particular == r.n_sub * r.te
    assert r.counters.interface_solves == r.te
