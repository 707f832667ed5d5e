"""Fine-solve error vs the oracle as a function of the PCG tolerance (developer tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from cases import rel_l2  # noqa: E402
from oracle_bind import oracle_lib  # noqa: E402
from paper_2103_11050_b200 import api, configs  # noqa: E402

name = sys.argv[1]
cfg = configs.build(name)
P = cfg.problem
o = api.Simulator(P, oracle_lib())
g = api.Simulator(P)
s = np.random.default_rng(11).uniform(0, 1, P.nx * P.ny)
kap = g.conductivity(s)
po, uo = o.fine_solve(kap)
pg, ug = g.fine_solve(kap)
print(os.environ.get("MPM2P_FINE_TOL", "1e-13"), g.fine_stats(), "p", rel_l2(pg, po), "u", rel_l2(ug, uo))

sys.path.insert(0, "tools")
from fine_pcg_proto import assemble  # noqa: E402

A, b = assemble(P.nx, P.ny, P.lx, P.ly, kap, np.asarray(P.bc.kind), np.asarray(P.bc.value))
bn = np.linalg.norm(b)
print("true relres: gpu", np.linalg.norm(b - A @ pg) / bn, "oracle", np.linalg.norm(b - A @ po) / bn)
