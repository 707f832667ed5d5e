"""Per-kernel device times (CUDA events around each launch) of one MRCM
rebuild (mrcm_solve) and one MPM-2P update of a config (developer tool)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2103_11050_b200 import api, configs
cfg = configs.build(sys.argv[1] if len(sys.argv) > 1 else "C5")
sim = api.Simulator(cfg.problem)
lib = sim.lib
kap = sim.conductivity(np.zeros(cfg.cells))
sim.mrcm_solve(kap)  # warm
prev = {}  # the report accumulates: subtract the previous totals
for what in ("rebuild", "mpm"):
    lib.profile_enable(sim.h, 1)
    lib.timer_record(sim.h, 0)
    if what == "rebuild":
        sim.mrcm_solve(kap)
    else:
        sim.mpm_pressure_update(kap * 1.01)
    lib.timer_record(sim.h, 1)
    ms = ctypes.c_double()
    lib.timer_elapsed(sim.h, 0, 1, ctypes.byref(ms))
    buf = ctypes.create_string_buffer(1 << 16)
    lib.profile_report(sim.h, buf, len(buf))
    lib.profile_enable(sim.h, 0)
    rows = []
    for line in buf.value.decode().splitlines():
        p = line.split()
        if len(p) == 3 and p[0] != "__launches__":
            t0, n0 = prev.get(p[0], (0.0, 0))
            prev[p[0]] = (float(p[2]), int(p[1]))
            if int(p[1]) > n0:
                rows.append((float(p[2]) - t0, p[0], int(p[1]) - n0))
    rows.sort(reverse=True)
    print(f"{cfg.name} {what}: {ms.value:.2f} ms total (events around every launch)")
    for t, k, n in rows[:14]:
        print(f"   {k:22s} {n:6d} launches {t:9.3f} ms")
