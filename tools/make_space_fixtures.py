#!/usr/bin/env python3
"""Oracle fixtures for the richer interface spaces at scale.

TEST INFRASTRUCTURE: runs the CPU oracle (oracle/liboracle.so) on the
BASELINE.json fields with the interface space swapped for the per-edge space
(H-bar = h), the linear space with adaptive alpha (the reference's
`high-contrast` preset, proj/src/config.cpp:474-475), the linear space alone,
adaptive alpha alone and the half-interface segments, over a short run, and
writes tests/golden/space_<case>.npz in tools/make_fixtures.py's format. The
interface system goes through the oracle's banded partial-pivot LU where the
dense LU of the reference would take minutes per rebuild (per-edge C2:
dim 15,360).

  python tools/make_space_fixtures.py                 # every case
  python tools/make_space_fixtures.py C2_edge C5_lin   # some
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

from paper_2103_11050_b200 import api  # noqa: E402
from make_fixtures import field_arrays, record_arrays  # noqa: E402
from space_cases import CASES, build_case  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def make(name):
    from oracle_bind import oracle_lib
    prob, split, s0, full, banded = build_case(name)
    if os.environ.get("EXTENDED") == "1":
        return make_extended(name, prob, split, s0, full, banded)
    lib = oracle_lib()
    lib.dll.oracle_set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
    lib.dll.oracle_set_interface_solver(2 if banded else 0)
    sim = api.Simulator(prob, lib)
    t0 = time.perf_counter()
    r = sim.run(split, s0)
    el = time.perf_counter() - t0
    sim.close()
    lib.dll.oracle_set_interface_solver(0)
    out = {"case": np.array(name), "split_te": np.array([split.te]), "oracle_seconds": np.array([el])}
    out.update(record_arrays(r))
    out.update(field_arrays(r, full=full))
    path = os.path.join(GOLDEN, f"space_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: te {r.record.te} rebuilds {r.record.update_steps} counters {r.record.counters}; "
          f"oracle {el:.1f} s -> {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


def make_extended(name, prob, split, s0, full, banded):
    """The same run in extended precision (liboracle_ld.so, long double), added
    to space_<name>.npz as ld_s / ld_p / ld_u (C5 cases: the ld_-prefixed sketch,
    subsample and non-zero saturations): the exact-answer yardstick where
    the double-precision oracle's own roundoff exceeds the 1e-8 bar (the C3 /
    C5 rule of tests/test_gpu_full_runs.py::check_fields_vs_truth)."""
    from oracle_bind import oracle_lib
    path = os.path.join(GOLDEN, f"space_{name}.npz")
    out = dict(np.load(path))
    lib = oracle_lib(True)
    lib.dll.oracle_set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
    lib.dll.oracle_set_interface_solver(2 if banded else 0)
    sim = api.Simulator(prob, lib)
    t0 = time.perf_counter()
    x = sim.run(split, s0)
    el = time.perf_counter() - t0
    sim.close()
    assert np.array_equal(np.array([s["rebuilt"] for s in x.record.steps], np.int8), out["rebuilt"])
    out.update(field_arrays(x, prefix="ld_", full=full))
    out["ld_seconds"] = np.array([el])
    np.savez_compressed(path, **out)
    print(f"{name} long double: {el:.0f} s -> {path}", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        make(n)
