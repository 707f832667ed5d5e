"""C5 early-step diagnostic (developer tool): GPU vs oracle (threaded) after
the initial MRCM solve and the first few Algorithm-1 steps, p / u / s errors
per step, and the same for a forced-alternative interface/repair path."""
import dataclasses
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2103_11050_b200 import api, configs  # noqa: E402
from oracle_bind import oracle_lib  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = configs.build("C5")
sp = dataclasses.replace(cfg.split, te=steps + 1)
o = oracle_lib()
o.dll.oracle_set_threads(os.cpu_count() or 1)
g = api.Simulator(cfg.problem)
x = api.Simulator(cfg.problem, o)
t0 = time.time()
g.run_begin(sp, cfg.s0())
x.run_begin(sp, cfg.s0())
print(f"begin {time.time() - t0:.1f} s", flush=True)


def rl(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for k in range(steps + 1):
    if k:
        g.run_step()
        x.run_step()
    sg, pg, ug = g.run_read()
    sx, px, ux = x.run_read()
    d = np.abs(ug - ux)
    i = int(np.argmax(d))
    print(f"step {k}: s {np.max(np.abs(sg - sx)):.3e} p {rl(pg, px):.3e} u {rl(ug, ux):.3e} "
          f"max|du| {d[i]:.3e} at face {i} (u {ux[i]:.3e}, |u|max {np.abs(ux).max():.3e})", flush=True)
