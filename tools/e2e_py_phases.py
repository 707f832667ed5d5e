"""Python-level wall phases of bench.py's end-to-end simulation (developer
tool): Simulator creation, mpm2p_run (uploads, steps, downloads), close."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_11050_b200 import api, configs
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.build(name)
lib = api.product_lib()
for rep in range(4):
    t0 = time.perf_counter()
    sim = api.Simulator(cfg.problem, lib)
    t1 = time.perf_counter()
    s0 = cfg.s0()
    t2 = time.perf_counter()
    res = sim.run(cfg.split, s0, cfg.inflow_sat)
    t3 = time.perf_counter()
    s, p, u = sim.run_read()
    t4 = time.perf_counter()
    sim.close()
    t5 = time.perf_counter()
    print(f"rep {rep}: Simulator {1e3*(t1-t0):.1f} ms  s0 {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f}  "
          f"extra download {1e3*(t4-t3):.1f}  close {1e3*(t5-t4):.1f}  rebuilds {res.record.tm_total}")
