#!/usr/bin/env python3
"""Generate the full-run oracle fixtures the GPU parity tests compare against.

TEST INFRASTRUCTURE: runs the CPU oracle (oracle/liboracle.so, the C++
restatement of the reference path) on the BASELINE.json configs exactly as
configs.build() defines them, and writes tests/golden/run_<name>.npz:

  per step   rebuilt (the MPM-2P vs MRCM decision sequence), dt, epsilon, pvi,
             cumulative basis-function counters
  per run    te, tm_total, breakthrough step / PVI, final PVI, SolveCounters,
             clamp count, max div ratio
  fields     final s, p, u. Full fields (C1-C4) are stored with the mantissa
             rounded to 32 bits (relative 2.3e-10, 40x below the 1e-8 parity
             bar) so they compress; C5 (16.8 M cells) stores a size-independent
             sketch instead: 64 seeded Rademacher projections of p and u
             (E[(r.d)^2] = |d|^2, so the sketch of a difference estimates its
             L2 norm), the norms, a seeded 1/256 subsample, and s at every cell
             where it is non-zero (the flood front has not reached the rest).

  python tools/make_fixtures.py C2 C3 C4          # full runs
  python tools/make_fixtures.py C5                # the whole C5 run (C5_STEPS=n: first n steps)

C3 is the two-pass run: to breakthrough b (stop_on_breakthrough), then
te = ceil(1.5 b) + 1; both passes are stored.
"""
from __future__ import annotations

import dataclasses
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2103_11050_b200 import api, configs  # noqa: E402
from golden_io import round_mantissa, sketch, subsample_idx  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
C5_STEPS = int(os.environ.get("C5_STEPS", "0"))  # 0: the whole run (see c5_split)


def record_arrays(res, prefix=""):
    st = res.record.steps
    rec = res.record
    c = rec.counters
    return {
        prefix + "rebuilt": np.array([s["rebuilt"] for s in st], np.int8),
        prefix + "dt": np.array([s["dt"] for s in st]),
        prefix + "epsilon": np.array([s["epsilon"] for s in st]),
        prefix + "pvi": np.array([s["pvi"] for s in st]),
        prefix + "bf_homog_cum": np.array([s["bf_homog_cum"] for s in st], np.int64),
        prefix + "bf_part_cum": np.array([s["bf_part_cum"] for s in st], np.int64),
        prefix + "meta_int": np.array([rec.te, rec.tm_total, rec.tm_updates, rec.breakthrough_step, c.homogeneous,
                                       c.particular, c.downscale, c.fine, c.interface_solves, rec.clamp_count,
                                       rec.repair_warnings], np.int64),
        prefix + "meta_f64": np.array([rec.breakthrough_pvi, rec.final_pvi, rec.max_div_ratio,
                                       rec.min_eps_margin]),
    }


def field_arrays(res, prefix="", full=True):
    if full:
        return {prefix + "s": round_mantissa(res.s_final), prefix + "p": round_mantissa(res.p_final),
                prefix + "u": round_mantissa(res.u_final)}
    out = {}
    for nm, x in (("p", res.p_final), ("u", res.u_final)):
        idx = subsample_idx(x.size)
        out[prefix + nm + "_sketch"] = sketch(x)
        out[prefix + nm + "_norm"] = np.array([np.linalg.norm(x)])
        out[prefix + nm + "_sub"] = x[idx]
    nz = np.flatnonzero(res.s_final)
    out[prefix + "s_nz_idx"] = nz.astype(np.int64)
    out[prefix + "s_nz_val"] = res.s_final[nz]
    return out


def c5_split(cfg):
    """The whole C5 run (te 501, the config's eta) unless C5_STEPS shortens it."""
    if not C5_STEPS:
        return cfg.split
    return dataclasses.replace(cfg.split, te=C5_STEPS + 1)


def run_oracle(cfg, split, extended=False):
    from oracle_bind import oracle_lib
    lib = oracle_lib(extended)
    # per-subdomain loops on all cores (bitwise the same result as 1 thread)
    lib.dll.oracle_set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
    sim = api.Simulator(cfg.problem, lib)
    t0 = time.perf_counter()
    r = sim.run(split, cfg.s0(), cfg.inflow_sat)
    el = time.perf_counter() - t0
    sim.close()
    return r, el


def make(name):
    cfg = configs.build(name)
    out = {"config": np.array(name)}
    if name == "C3":
        r1, t1 = run_oracle(cfg, cfg.split)
        b = r1.record.breakthrough_step
        assert b >= 0, "C3 pass 1 did not break through"
        te2 = configs.breakthrough_plus_50(b)
        sp2 = dataclasses.replace(cfg.split, stop_on_breakthrough=False, te=te2)
        r2, t2 = run_oracle(cfg, sp2)
        out.update(record_arrays(r1, "pass1_"))
        out.update(field_arrays(r1, "pass1_"))
        out.update(record_arrays(r2))
        out.update(field_arrays(r2))
        out["split_te"] = np.array([te2])
        # the same two passes in extended precision (long double): the exact
        # answer to ~1e-10, the yardstick for double-precision roundoff on this
        # ill-conditioned config (K spans 1.6e7, cond(M) ~ 2e9)
        x1, t3 = run_oracle(cfg, cfg.split, extended=True)
        x2, t4 = run_oracle(cfg, sp2, extended=True)
        assert x1.record.breakthrough_step == b and x2.record.te == r2.record.te
        for pre, x, r in (("pass1_", x1, r1), ("", x2, r2)):
            assert [s["rebuilt"] for s in x.record.steps] == [s["rebuilt"] for s in r.record.steps]
            out[pre + "ld_s"] = round_mantissa(x.s_final)
            out[pre + "ld_p"] = round_mantissa(x.p_final)
            out[pre + "ld_u"] = round_mantissa(x.u_final)
            out[pre + "ld_dt"] = np.array([s["dt"] for s in x.record.steps])
            out[pre + "ld_pvi"] = np.array([s["pvi"] for s in x.record.steps])
        el = t1 + t2
        msg = (f"pass1 te {r1.record.te} (breakthrough {b}), pass2 te {r2.record.te} rebuilds {r2.record.tm_total}; "
               f"long double {t3 + t4:.0f} s")
    elif name == "C5":
        sp = c5_split(cfg)
        if os.environ.get("EXTENDED") == "1":
            # the whole run in extended precision (long double), the exact-answer
            # yardstick for double-precision roundoff at C5 (written beside run_C5.npz)
            x, el = run_oracle(cfg, sp, extended=True)
            out.update(record_arrays(x))
            out.update(field_arrays(x, full=False))
            path = os.path.join(GOLDEN, "run_C5_ld.npz")
            np.savez_compressed(path, **out)
            print(f"C5 long double: rebuilds {x.record.update_steps}; {el:.0f} s -> {path}", flush=True)
            return
        r, el = run_oracle(cfg, sp)
        out.update(record_arrays(r))
        out.update(field_arrays(r, full=False))
        out["split_te"] = np.array([sp.te])
        msg = f"te {r.record.te} rebuild steps {r.record.update_steps}"
    else:
        r, el = run_oracle(cfg, cfg.split)
        out.update(record_arrays(r))
        out.update(field_arrays(r))
        out["split_te"] = np.array([cfg.split.te])
        msg = f"te {r.record.te} rebuilds {r.record.tm_total}"
    out["oracle_seconds"] = np.array([el])
    path = os.path.join(GOLDEN, f"run_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {msg}; oracle {el:.1f} s -> {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C2", "C3", "C4"]:
        make(n.upper())
