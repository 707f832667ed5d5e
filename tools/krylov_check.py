"""K7 check (developer tool): MINRES interface solve vs the dense inverse and
the oracle; prints iteration counts and wall times. Usage:
    python tools/krylov_check.py [small|C2|C5] ...
"""
import dataclasses
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2103_11050_b200 import api, configs  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def sim(prob, mode):
    os.environ["MPM2P_IFACE"] = mode
    try:
        return api.Simulator(prob)
    finally:
        os.environ.pop("MPM2P_IFACE", None)


def small():
    from cases import problem, random_kappa
    from oracle_bind import oracle_lib
    O = oracle_lib()
    nx = ny = 32
    for (nsx, nsy, sp, hb, contrast) in [(4, 4, 0, 0, 10.0), (4, 4, 1, 0, 10.0), (2, 4, 0, 1, 100.0), (8, 8, 0, 0, 1e3)]:
        K = random_kappa(nx, ny, 1, 1.0 / contrast, 1.0)
        prob = problem(nx, ny, nsx, nsy, K, M=5.0, space=sp, hbar=hb)
        g, o = sim(prob, "krylov"), api.Simulator(prob, O)
        sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
        kn = K * np.exp(0.05 * np.random.default_rng(3).standard_normal(K.size))
        mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
        print(f"small {nsx}x{nsy} sp={sp} hb={hb} contrast={contrast:g}: coeffs {rel(sg.coeffs, so.coeffs):.2e} "
              f"p {rel(sg.p, so.p):.2e} u {rel(sg.u, so.u):.2e} mpm p {rel(mg.p, mo.p):.2e} u {rel(mg.u, mo.u):.2e}",
              flush=True)


def full(name, te):
    cfg = configs.build(name)
    sp = dataclasses.replace(cfg.split, te=te) if te else cfg.split
    out = {}
    for mode in (["dense", "krylov"] if name != "C5" else ["krylov"]):
        s = sim(cfg.problem, mode)
        t0 = time.time()
        r = s.run(sp, cfg.s0(), cfg.inflow_sat)
        t1 = time.time()
        rec = r.record
        out[mode] = r
        print(f"{name} {mode}: te={rec.te} tm={rec.tm_total} wall={t1 - t0:.2f}s krylov={rec.interface_krylov} "
              f"iters total={rec.interface_iterations} max={rec.interface_max_iterations} "
              f"pvi={rec.final_pvi:.6f} maxdiv={rec.max_div_ratio:.2e}", flush=True)
    if len(out) == 2:
        a, b = out["dense"], out["krylov"]
        print(f"{name} krylov vs dense: s {rel(b.s_final, a.s_final):.2e} p {rel(b.p_final, a.p_final):.2e} "
              f"u {rel(b.u_final, a.u_final):.2e} updates {a.record.update_steps == b.record.update_steps}", flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["small"]:
        if arg == "small":
            small()
        else:
            nm, _, te = arg.partition(":")
            full(nm, int(te) if te else 0)
