import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_11050_b200 import api, configs
import dataclasses
cfg = configs.build(sys.argv[1] if len(sys.argv) > 1 else "C2")
sim = api.Simulator(cfg.problem)
sp = dataclasses.replace(cfg.split, te=6)
sim.run_begin(sp, cfg.s0(), cfg.inflow_sat)
while sim.run_step() is not None:
    pass
print("ok", sim.run_end().tm_total)
