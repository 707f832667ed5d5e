"""Iterations and wall time of the device fine solve on the configs (developer tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2103_11050_b200 import api, configs  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    cfg = configs.build(name)
    sim = api.Simulator(cfg.problem)
    rng = np.random.default_rng(1)
    s = rng.uniform(0, 1, cfg.cells)
    kap = sim.conductivity(s)
    sim.fine_solve(kap)
    t = time.perf_counter()
    reps = 3
    for _ in range(reps):
        sim.fine_solve(kap)
    dt = (time.perf_counter() - t) / reps
    it, rr, dres, dsc = sim.fine_stats()
    print(f"{name}: {dt * 1e3:.2f} ms per cold fine solve, {it} PCG iterations, relres {rr:.2e}, div {dres / dsc:.2e}")
    sim.close()
