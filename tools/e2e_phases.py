"""Wall-time phases of one end-to-end simulation through the C ABI (developer tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_11050_b200 import api, configs
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.build(name)
lib = api.product_lib()
for rep in range(3):
    t0 = time.perf_counter()
    sim = api.Simulator(cfg.problem, lib)
    t1 = time.perf_counter()
    sim.run_begin(cfg.split, cfg.s0(), cfg.inflow_sat)
    t2 = time.perf_counter()
    n = 0
    marks = []
    while True:
        ts = time.perf_counter()
        r = sim.run_step()
        if r is None:
            break
        n += 1
        if n <= 3 or r["rebuilt"] and len(marks) < 6:
            marks.append((n, r["rebuilt"], round(1e3 * (time.perf_counter() - ts), 2)))
    t3 = time.perf_counter()
    rec = sim.run_end()
    t35 = time.perf_counter()
    sim.close()
    t4 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms  begin {1e3*(t2-t1):.1f} ms  {n} steps {1e3*(t3-t2):.1f} ms "
          f"({1e3*(t3-t2)/max(n,1):.3f} ms/step)  run_end {1e3*(t35-t3):.1f} ms  close {1e3*(t4-t35):.1f} ms  "
          f"rebuilds {rec.tm_total}", flush=True)
