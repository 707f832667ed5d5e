"""Richer interface spaces at scale: feasibility and timing of
per-edge / linear / adaptive-alpha spaces on the C2 / C4 / C5 fields, GPU only.
Usage (GPU box): python tools/spaces_probe.py [C2 C4 C5 ...]"""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_11050_b200 import api, configs  # noqa: E402

CASES = {
    "C2": [("per-edge", dict(hbar_mode=api.HBAR_PER_EDGE)),
           ("linear+adaptive", dict(space_kind=api.SPACE_LINEAR, alpha=api.AlphaSpec(mode=api.ALPHA_ADAPTIVE)))],
    "C4": [("per-edge", dict(hbar_mode=api.HBAR_PER_EDGE)),
           ("linear+adaptive", dict(space_kind=api.SPACE_LINEAR, alpha=api.AlphaSpec(mode=api.ALPHA_ADAPTIVE)))],
    "C5": [("linear", dict(space_kind=api.SPACE_LINEAR)),
           ("adaptive", dict(alpha=api.AlphaSpec(mode=api.ALPHA_ADAPTIVE))),
           ("half", dict(hbar_mode=api.HBAR_HALF))],
}


def main():
    names = sys.argv[1:] or list(CASES)
    steps = int(os.environ.get("PROBE_STEPS", "21"))
    for name in names:
        cfg = configs.build(name, te_override=steps)
        for label, kw in CASES[name]:
            prob = dataclasses.replace(cfg.problem, **kw)
            t0 = time.perf_counter()
            try:
                sim = api.Simulator(prob)
            except Exception as e:  # noqa: BLE001
                print(f"{name} {label}: create failed: {type(e).__name__}: {e}", flush=True)
                continue
            t1 = time.perf_counter()
            try:
                res = sim.run(cfg.split, s0=cfg.s0())
            except Exception as e:  # noqa: BLE001
                print(f"{name} {label}: run failed: {type(e).__name__}: {e}", flush=True)
                sim.close()
                continue
            t2 = time.perf_counter()
            rec = res.record
            reb = sum(s["rebuilt"] for s in rec.steps)
            ok = bool(np.all(np.isfinite(res.u_final)))
            print(f"{name} {label}: create {t1 - t0:.2f}s run {t2 - t1:.2f}s steps {len(rec.steps)} rebuilds {reb} "
                  f"finite {ok} counters {rec.counters}", flush=True)
            sim.close()


if __name__ == "__main__":
    main()
