"""Per-step trace of the ping-pong Gauss-Jordan (MPM2P_GJ_TRACE=1) on one
rebuild of a config (developer tool)."""
import os, sys
os.environ["MPM2P_GJ_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2103_11050_b200 import api, configs
cfg = configs.build(sys.argv[1] if len(sys.argv) > 1 else "C2")
sim = api.Simulator(cfg.problem)
kap = sim.conductivity(np.zeros(cfg.cells))
for _ in range(2):
    sim.mrcm_solve(kap)
