import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle_bind import oracle_lib
from paper_2103_11050_b200 import api, configs
from cases import rel_l2
O = oracle_lib()
c = configs.build("C3")
g, o = api.Simulator(c.problem), api.Simulator(c.problem, O)
kap = o.conductivity(np.zeros(c.cells))
sg, so = g.mrcm_solve(kap), o.mrcm_solve(kap)
M = o.interface_matrix()
print("M diff", rel_l2(g.interface_matrix(), M))
print("coeffs", rel_l2(sg.coeffs, so.coeffs), "p", rel_l2(sg.p, so.p), "u", rel_l2(sg.u, so.u))
# residual of each coefficient vector against the oracle's M and the oracle's rhs (M @ so.coeffs)
b = M @ so.coeffs
print("resid gpu", np.linalg.norm(M @ sg.coeffs - b) / np.linalg.norm(b))
xt = np.linalg.solve(M, b)
print("numpy vs oracle", rel_l2(xt, so.coeffs), "numpy vs gpu", rel_l2(xt, sg.coeffs))
rng = np.random.default_rng(1)
for amp in (0.0, 0.05):
    kn = kap * np.exp(amp * rng.standard_normal(kap.size))
    mg, mo = g.mpm_pressure_update(kn), o.mpm_pressure_update(kn)
    print("mpm amp", amp, "coeffs", rel_l2(mg.coeffs, mo.coeffs), "p", rel_l2(mg.p, mo.p), "u", rel_l2(mg.u, mo.u))
