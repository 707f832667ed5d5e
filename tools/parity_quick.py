"""Quick GPU-vs-oracle parity sweep (developer tool; prints one line per check)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2103_11050_b200 import api  # noqa: E402
from cases import problem, random_kappa, rel_l2  # noqa: E402
from oracle_bind import oracle_lib  # noqa: E402

O = oracle_lib()


def both(prob):
    return api.Simulator(prob), api.Simulator(prob, O)


def check(name, v, tol):
    ok = v <= tol
    print(f"[{'PASS' if ok else 'FAIL'}] {name}: {v:.3e} (tol {tol:g})", flush=True)
    return ok


def main():
    ok = True
    # transport
    nx = ny = 32
    K = random_kappa(nx, ny, 1)
    g, o = both(problem(nx, ny, 4, 4, K, M=5.0))
    sol = o.mrcm_solve(K)
    u = sol.u
    rng = np.random.default_rng(3)
    s = rng.uniform(0, 1, nx * ny)
    ok &= check("conductivity bitwise", np.max(np.abs(g.conductivity(s) - o.conductivity(s))), 0.0)
    ok &= check("max slope bitwise", abs(g.max_fractional_flow_slope() - o.max_fractional_flow_slope()), 0.0)
    dtg, dto = g.cfl_timestep(u, 0.9, 1.0), o.cfl_timestep(u, 0.9, 1.0)
    ok &= check("cfl bitwise", abs(dtg - dto), 0.0)
    sg, so = g.upwind_step(s, 1.0, u, dto), o.upwind_step(s, 1.0, u, dto)
    ok &= check("upwind bitwise", np.max(np.abs(sg - so)), 0.0)
    ok &= check("injection", abs(g.injection_rate(u, 1.0) - o.injection_rate(u, 1.0)), 0.0)
    ok &= check("outlet", abs(g.max_outlet_saturation(s, u) - o.max_outlet_saturation(s, u)), 0.0)
    kn = K * 1.01
    ok &= check("epsilon", abs(g.epsilon(kn, K) - o.epsilon(kn, K)) / o.epsilon(kn, K), 1e-14)
    bg, bo = g.compute_beta(K), o.compute_beta(K)
    ok &= check("beta bitwise", max(np.max(np.abs(bg[0] - bo[0])), np.max(np.abs(bg[1] - bo[1]))), 0.0)
    # mrcm
    for (nsx, nsy, sp, hb, M) in [(4, 4, 0, 0, 5.0), (2, 2, 0, 1, 5.0), (4, 4, 1, 0, 5.0), (2, 4, 0, 0, 5.0)]:
        prob = problem(nx, ny, nsx, nsy, K, M=M, space=sp, hbar=hb)
        g, o = both(prob)
        t0 = time.time()
        sg = g.mrcm_solve(K)
        t1 = time.time()
        so = o.mrcm_solve(K)
        name = f"mrcm {nsx}x{nsy} space={sp} hbar={hb}"
        ok &= check(name + " M", rel_l2(g.interface_matrix(), o.interface_matrix()), 1e-12)
        ok &= check(name + " coeffs", rel_l2(sg.coeffs, so.coeffs), 1e-9)
        ok &= check(name + " p", rel_l2(sg.p, so.p), 1e-9)
        ok &= check(name + " u", rel_l2(sg.u, so.u), 1e-9)
        ok &= check(name + " counters", float(sg.counters != so.counters), 0)
        kn = K * np.exp(0.05 * rng.standard_normal(K.size))
        mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
        ok &= check(name + " mpm p", rel_l2(mg.p, mo.p), 1e-9)
        ok &= check(name + " mpm u", rel_l2(mg.u, mo.u), 1e-9)
        ok &= check(name + " mpm counters", float(mg.counters != mo.counters), 0)
        print(f"   gpu mrcm_solve wall {1e3*(t1-t0):.1f} ms")
    # full runs
    for (nsx, nsy, eta, mode, meth) in [(4, 4, 0.01, api.EPS_RELATIVE, api.MPM2P),
                                         (4, 4, 0.01, api.EPS_MOBILITY, api.MPM2P),
                                         (4, 4, 0.01, api.EPS_RELATIVE, api.MRCM_EVERY_STEP)]:
        nx = ny = 64
        K = random_kappa(nx, ny, 7, 0.1, 10.0)
        prob = problem(nx, ny, nsx, nsy, K, M=5.0)
        g, o = both(prob)
        sp = api.SplittingConfig(method=meth, eta=eta, eta_mode=mode, te=60, cfl_safety=0.5)
        t0 = time.time()
        rg = g.run(sp)
        t1 = time.time()
        ro = o.run(sp)
        t2 = time.time()
        name = f"run {nx}x{ny}/{nsx}x{nsy} mode={mode} meth={meth}"
        seq_g = [s["rebuilt"] for s in rg.record.steps]
        seq_o = [s["rebuilt"] for s in ro.record.steps]
        ok &= check(name + " decisions", float(seq_g != seq_o), 0)
        ok &= check(name + " s", np.max(np.abs(rg.s_final - ro.s_final)), 1e-8)
        ok &= check(name + " p", rel_l2(rg.p_final, ro.p_final), 1e-8)
        ok &= check(name + " u", rel_l2(rg.u_final, ro.u_final), 1e-8)
        print(f"   rebuilds {rg.record.tm_total}/{ro.record.tm_total} margin {rg.record.min_eps_margin:.3e} "
              f"gpu {1e3*(t1-t0):.0f} ms cpu {1e3*(t2-t1):.0f} ms")
    print("ALL PASS" if ok else "SOME FAILED")


if __name__ == "__main__":
    main()
