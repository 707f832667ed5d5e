"""Short C2 workload for ncu: two rebuilds (mrcm_solve) and two MPM updates."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2103_11050_b200 import api, configs
cfg = configs.build(sys.argv[1] if len(sys.argv) > 1 else "C2")
sim = api.Simulator(cfg.problem)
kap = sim.conductivity(np.zeros(cfg.cells))
for _ in range(2):
    sim.mrcm_solve(kap)
for _ in range(2):
    sim.mpm_pressure_update(kap * 1.01)
print("ok")
