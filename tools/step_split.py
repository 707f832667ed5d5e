"""Device time per Algorithm-1 step split by branch (MPM-2P reuse vs MRCM
rebuild), with and without an L2 flush before each step (developer tool)."""
import ctypes, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_11050_b200 import api, configs
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
cfg = configs.build(name)
lib = api.product_lib()
import dataclasses
split = dataclasses.replace(cfg.split, stop_on_breakthrough=False, te=max(cfg.split.te or 0, 2 * nsteps + 10))
sim = api.Simulator(cfg.problem, lib)
sim.run_begin(split, cfg.s0(), cfg.inflow_sat)
for _ in range(5):
    sim.run_step()
for flush in (1, 0):
    t = {0: [], 1: []}
    for _ in range(nsteps):
        if flush:
            lib.flush_l2(sim.h)
        lib.timer_record(sim.h, 0)
        r = sim.run_step()
        lib.timer_record(sim.h, 1)
        if r is None:
            break
        ms = ctypes.c_double()
        lib.timer_elapsed(sim.h, 0, 1, ctypes.byref(ms))
        t[r["rebuilt"]].append(ms.value * 1e3)
    for b, nm in ((0, "mpm"), (1, "rebuild")):
        v = t[b]
        if v:
            print(f"{name} flush={flush} {nm:8s} n={len(v):4d} median {statistics.median(v):8.1f} us "
                  f"mean {statistics.mean(v):8.1f} us min {min(v):8.1f} us")
sim.run_end()
sim.close()
if os.environ.get("MPM2P_GRAPH_TIMING") == "1":  # replay-only device time (timers 14/15 inside run_step)
    sim = api.Simulator(cfg.problem, lib)
    sim.run_begin(split, cfg.s0(), cfg.inflow_sat)
    t = {0: [], 1: []}
    for _ in range(nsteps):
        lib.flush_l2(sim.h)
        r = sim.run_step()
        if r is None:
            break
        ms = ctypes.c_double()
        lib.timer_elapsed(sim.h, 14, 15, ctypes.byref(ms))
        t[r["rebuilt"]].append(ms.value * 1e3)
    for b, nm in ((0, "mpm"), (1, "rebuild")):
        v = t[b][2:] if b == 0 else t[b]
        if v:
            print(f"{name} replay-only {nm:8s} n={len(v):4d} median {statistics.median(v):8.1f} us")
    sim.run_end()
    sim.close()
