"""The MRCM sub-step entry points (proj/include/mrcmflow/mrcm.hpp:77-136,
157-161) through the C ABI: compute_basis_set, restrict_physical_data,
solve_particular, solve_interface, reconstruct, averaged_skeleton_flux,
downscale and weak_continuity_residuals, each against the oracle's
restatement of the same reference function on the same inputs, and composed
into mrcm_solve (mrcm.cpp:440-457)."""
import numpy as np
import pytest

from cases import problem, random_kappa, rel_l2
from paper_2103_11050_b200 import api


CASES = {
    "c1like": dict(nx=64, ny=64, nsx=4, nsy=4, bc="pd", space=api.SPACE_CONSTANT, hbar=api.HBAR_WHOLE),
    "linear": dict(nx=48, ny=32, nsx=3, nsy=2, bc="ui", space=api.SPACE_LINEAR, hbar=api.HBAR_WHOLE),
    "half_robin": dict(nx=64, ny=32, nsx=4, nsy=2, bc="robin", space=api.SPACE_CONSTANT, hbar=api.HBAR_HALF),
    "wide32": dict(nx=96, ny=64, nsx=3, nsy=2, bc="pd", space=api.SPACE_CONSTANT, hbar=api.HBAR_WHOLE),
}


def _bc(name, nx, ny):
    if name == "pd":
        return api.pressure_drop(nx, ny)
    if name == "ui":
        return api.unit_inflow(nx, ny)
    return api.BoundarySpec.uniform(nx, ny, (api.ROBIN, 0.5, 1.0), (api.PRESSURE, 0.0), (api.FLUX, 0.0),
                                    (api.ROBIN, 2.0, 0.0))


def _pair(oracle, case):
    c = CASES[case]
    K = random_kappa(c["nx"], c["ny"], 17, 0.05, 20.0)
    prob = problem(c["nx"], c["ny"], c["nsx"], c["nsy"], K, bc=_bc(c["bc"], c["nx"], c["ny"]), space=c["space"],
                   hbar=c["hbar"])
    return api.Simulator(prob), api.Simulator(prob, oracle), K


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_substeps_match_oracle(oracle, case):
    g, o, K = _pair(oracle, case)
    assert g.sizes.sub_faces == o.sizes.sub_faces
    cg, co = g.compute_basis_set(K), o.compute_basis_set(K)
    assert cg == co
    # restrict_physical_data: indexing and copies, bit-exact
    dg, do = g.restrict_physical_data(), o.restrict_physical_data()
    for k in ("q", "kind", "value", "beta", "robin_rhs"):
        assert np.array_equal(dg[k], do[k]), k
    # solve_particular on the same data: exact direct solves on both sides
    pg, cpg = g.solve_particular(do)
    po, cpo = o.solve_particular(do)
    assert cpg == cpo and cpg.particular == g.sizes.n_sub
    for k in ("p", "u", "boundary_p"):
        assert rel_l2(pg[k], po[k]) < 1e-10, k
    # solve_interface on the oracle's particular solution
    xg, cig = g.solve_interface(po)
    xo, cio = o.solve_interface(po)
    assert cig.interface_solves == cio.interface_solves == 1
    if g.dim:
        assert rel_l2(xg, xo) < 1e-9
    # reconstruct with the same coefficients and particular solution
    rg, ro = g.reconstruct(xo, po), o.reconstruct(xo, po)
    for k in ("p", "u", "boundary_p"):
        assert rel_l2(rg[k], ro[k]) < 1e-11, k
    # averaged_skeleton_flux: 0.5 (u_minus + u_plus), bitwise
    fg, fo = g.averaged_skeleton_flux(ro), o.averaged_skeleton_flux(ro)
    assert np.array_equal(fg, fo)
    # downscale of the same reconstruction and skeleton flux
    kn = K * 1.1
    ug = g.downscale(kn, ro, fo)
    uo = o.downscale(kn, ro, fo)
    assert rel_l2(ug[0], uo[0]) < 1e-9 and rel_l2(ug[1], uo[1]) < 1e-9
    assert ug[3].downscale == uo[3].downscale == g.sizes.n_sub
    assert abs(ug[2].repair_max - uo[2].repair_max) <= 1e-9 * max(uo[2].flux_scale, 1.0)
    assert ug[2].repair_warning == uo[2].repair_warning
    # weak continuity residuals of the reconstruction (both ~0 for a converged solve)
    wg, wo = g.weak_continuity_residuals(ro), o.weak_continuity_residuals(ro)
    scale = max(np.max(np.abs(ro["u"])), np.max(np.abs(ro["boundary_p"])), 1.0)
    for a, b in zip(wg, wo):
        assert abs(a - b) <= 1e-9 * scale


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_substeps_compose_to_mrcm_solve(oracle, case):
    """compute_basis_set -> restrict -> solve_particular -> solve_interface ->
    reconstruct -> averaged_skeleton_flux -> downscale reproduces mrcm_solve
    (mrcm.cpp:440-457) on the device, and the weak jumps of its
    reconstruction vanish (mrcm.hpp:155-161)."""
    g, o, K = _pair(oracle, case)
    ref = g.mrcm_solve(K)
    g.compute_basis_set(K)
    part, _ = g.solve_particular(g.restrict_physical_data())
    co, _ = g.solve_interface(part)
    recon = g.reconstruct(co, part)
    flux = g.averaged_skeleton_flux(recon)
    p, u, info, cnt = g.downscale(K, recon, flux)
    assert rel_l2(p, ref.p) < 1e-10 and rel_l2(u, ref.u) < 1e-10
    if g.dim:
        assert rel_l2(co, ref.coeffs) < 1e-10
    fj, pj = g.weak_continuity_residuals(recon)
    scale = max(np.max(np.abs(recon["u"])), np.max(np.abs(recon["boundary_p"])), 1.0)
    assert fj <= 1e-8 * scale and pj <= 1e-8 * scale
    mo = o.mrcm_solve(K)
    assert rel_l2(u, mo.u) < 1e-8


@pytest.mark.gpu
def test_solve_particular_structure_check(oracle):
    """elliptic.cpp:155-160: a solve whose boundary kinds or Robin betas differ
    from the factorization's raises NumericError."""
    g, o, K = _pair(oracle, "c1like")
    for sim in (g, o):
        sim.compute_basis_set(K)
        d = sim.restrict_physical_data()
        bad = dict(d)
        bad["beta"] = d["beta"] * np.where(d["kind"] == api.ROBIN, 1.5, 1.0)
        with pytest.raises(api.NumericError):
            sim.solve_particular(bad)
        bad = dict(d)
        k = d["kind"].copy()
        k[0, 0] = api.FLUX if k[0, 0] != api.FLUX else api.PRESSURE
        bad["kind"] = k
        with pytest.raises(api.NumericError):
            sim.solve_particular(bad)


@pytest.mark.gpu
def test_substeps_need_a_basis(oracle):
    g, o, K = _pair(oracle, "c1like")
    for sim in (g, o):
        with pytest.raises(api.ConfigError):
            sim.restrict_physical_data()


def _snap_run(sim, split, steps):
    got = {}
    res = sim.run(split, snapshot_steps=steps, snap=lambda n, s, p, u: got.__setitem__(n, (s, p, u)))
    return res, got


@pytest.mark.parametrize("gpu", [pytest.param(True, marks=pytest.mark.gpu),
                                 False])
def test_run_snapshots(oracle, gpu):
    """run(in, snapshot_steps, snap) (simulation.hpp:119-128, simulation.cpp:
    224-226): the callback fires once per listed step (0 = the initial solve)
    with the fields the step-by-step driver holds after that step."""
    nx = ny = 32
    K = random_kappa(nx, ny, 4, 0.1, 10.0)
    prob = problem(nx, ny, 4, 4, K)
    sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, te=12, cfl_safety=0.5)
    make = (lambda: api.Simulator(prob)) if gpu else (lambda: api.Simulator(prob, oracle))
    want = [0, 3, 7, 11, 50]
    res, got = _snap_run(make(), sp, want)
    assert sorted(got) == [0, 3, 7, 11]
    ref = make()
    ref.run_begin(sp)
    for n in range(0, 12):
        if n > 0:
            assert ref.run_step() is not None
        if n in got:
            s, p, u = ref.run_read()
            assert np.array_equal(got[n][0], s) and np.array_equal(got[n][1], p) and np.array_equal(got[n][2], u)
    plain = make().run(sp)
    assert np.array_equal(plain.s_final, res.s_final) and np.array_equal(plain.u_final, res.u_final)
    if gpu:
        _, go = _snap_run(api.Simulator(prob, oracle), sp, want)
        for n in got:
            assert np.max(np.abs(got[n][0] - go[n][0])) <= 1e-8 and rel_l2(got[n][2], go[n][2]) <= 1e-8
