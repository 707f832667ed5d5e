import os, sys, time
sys.path.insert(0, "/root/repo")
from paper_2103_11050_b200 import api, configs
cfg = configs.build("C2")
lib = api.product_lib()
s = api.Simulator(cfg.problem, lib); s.close()
for rep in range(5):
    t0 = time.perf_counter()
    sim = api.Simulator(cfg.problem, lib)
    t1 = time.perf_counter()
    res = sim.run(cfg.split, cfg.s0(), cfg.inflow_sat)
    t2 = time.perf_counter()
    sim.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} run {1e3*(t2-t1):.1f} close {1e3*(t3-t2):.1f} total {1e3*(t3-t0):.1f} ms", flush=True)
