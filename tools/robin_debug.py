"""Developer probe: GPU vs oracle MPM-2P update with physical Robin faces,
per subdomain, under the kernel-variant switches."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from cases import problem, random_kappa, rel_l2  # noqa: E402
from oracle_bind import oracle_lib  # noqa: E402
from paper_2103_11050_b200 import api  # noqa: E402

nx, ny = 48, 32
K = random_kappa(nx, ny, 21, 0.1, 10.0)
sides = {
    "all": ((api.ROBIN, 0.5, 1.0), (api.ROBIN, 2.0, -0.5), (api.ROBIN, 1.0, 0.25), (api.ROBIN, 0.3, 0.0)),
    "all_rhs0": ((api.ROBIN, 0.5, 0.0), (api.ROBIN, 2.0, 0.0), (api.ROBIN, 1.0, 0.0), (api.ROBIN, 0.3, 0.0)),
    "w_e": ((api.ROBIN, 0.5, 1.0), (api.ROBIN, 2.0, -0.5), (api.FLUX, 0.0), (api.FLUX, 0.0)),
    "w_p": ((api.ROBIN, 0.5, 1.0), (api.PRESSURE, 0.0), (api.FLUX, 0.0), (api.FLUX, 0.0)),
    "s_p": ((api.PRESSURE, 1.0), (api.PRESSURE, 0.0), (api.ROBIN, 1.0, 0.25), (api.FLUX, 0.0)),
    "flux_p": ((api.FLUX, -1.0), (api.PRESSURE, 0.0), (api.FLUX, 0.0), (api.FLUX, 0.0)),
}
o = oracle_lib()
for name, sd in sides.items():
    bc = api.BoundarySpec.uniform(nx, ny, *sd)
    prob = problem(nx, ny, 4, 4, K, bc=bc)
    g, r = api.Simulator(prob), api.Simulator(prob, o)
    sg, so = g.mrcm_solve(K), r.mrcm_solve(K)
    out = [f"mrcm p {rel_l2(sg.p, so.p):.1e} u {rel_l2(sg.u, so.u):.1e}"]
    for amp in (0.0, 0.1):
        kn = K * np.exp(amp * np.random.default_rng(4).standard_normal(K.size))
        mg, mo = g.mpm_pressure_update(kn), r.mpm_pressure_update(kn)
        out.append(f"mpm{amp} p {rel_l2(mg.p, mo.p):.1e} u {rel_l2(mg.u, mo.u):.1e} co {rel_l2(mg.coeffs, mo.coeffs):.1e}")
    print(os.environ.get("TAG", ""), name, "; ".join(out), flush=True)
