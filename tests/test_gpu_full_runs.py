"""Full-run parity of every BASELINE.json config against committed oracle fixtures.

north_star: every config matches the CPU oracle after the FULL run —
decision sequence (MPM-2P vs MRCM) bit-exact, SolveCounters exact, p and u
relative L2 <= 1e-8, s max-abs <= 1e-8. The fixtures under tests/golden/ were
written by tools/make_fixtures.py, which runs the oracle (the C++ restatement
of the reference path, oracle/) on exactly configs.build(name):

  C1  201 steps       (also run live against the oracle in test_gpu_parity.py)
  C2  2,001 steps     126 MRCM rebuilds
  C3  two passes: to breakthrough (oracle: step 5,501), then te = ceil(1.5 b) + 1
  C4  5,001 steps
  C5  501 steps on 4096^2 cells, 16,384 subdomains (oracle with the banded
      interface LU; fields compared through a seeded random-projection sketch)

Full fields are stored with 32-bit mantissas (relative rounding 2.3e-10), far
below the 1e-8 bar; the tests charge that rounding to the tolerance explicitly.
"""
import dataclasses
import os

import numpy as np
import pytest

from paper_2103_11050_b200 import api, configs

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL_PU = 1e-8
TOL_S = 1e-8
FIXTURE_ROUNDING = 2.0 ** -32  # relative rounding of the stored fields (tools/make_fixtures.py)


def load(name):
    path = os.path.join(GOLDEN, f"run_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path}: run tools/make_fixtures.py {name}")
    return dict(np.load(path))


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check_record(run, fx, prefix="", exact_yardstick=False):
    rec = run.record
    rebuilt = np.array([s["rebuilt"] for s in rec.steps], np.int8)
    exp = fx[prefix + "rebuilt"]
    assert rebuilt.shape == exp.shape, (rebuilt.shape, exp.shape)
    diff = np.flatnonzero(rebuilt != exp)
    assert diff.size == 0, f"decision sequence differs first at step {diff[:5]}"
    c = rec.counters
    got = [rec.te, rec.tm_total, rec.tm_updates, rec.breakthrough_step, c.homogeneous, c.particular,
           c.downscale, c.fine, c.interface_solves]
    assert got == list(fx[prefix + "meta_int"][:9]), (got, fx[prefix + "meta_int"][:9])
    for key in ("bf_homog_cum", "bf_part_cum"):
        assert np.array_equal(np.array([s[key] for s in rec.steps]), fx[prefix + key]), key
    for key in ("dt", "pvi"):
        got = np.array([s[key] for s in rec.steps])
        ref = fx[prefix + key]
        den = np.maximum(np.abs(ref), 1e-300)
        d_go = float(np.max(np.abs(got - ref) / den))
        if d_go <= 1e-8 or not exact_yardstick:
            assert d_go <= 1e-8, (key, d_go)
            continue
        # dt comes from the velocity field (CFL), so on an ill-conditioned config
        # it carries u's roundoff: compare with the oracle's distance to the
        # extended-precision run, as for the fields
        ext = fx[prefix + "ld_" + key]
        d_gx = float(np.max(np.abs(got - ext) / den))
        d_ox = float(np.max(np.abs(ref - ext) / den))
        assert d_gx <= max(1e-8, 3.0 * d_ox), (key, {"gpu_vs_oracle": d_go, "gpu_vs_exact": d_gx,
                                                      "oracle_vs_exact": d_ox})


def check_fields(run, fx, prefix=""):
    ds = float(np.max(np.abs(run.s_final - fx[prefix + "s"])))
    dp = rel_l2(run.p_final, fx[prefix + "p"])
    du = rel_l2(run.u_final, fx[prefix + "u"])
    assert ds <= TOL_S + FIXTURE_ROUNDING, ds
    assert dp <= TOL_PU + FIXTURE_ROUNDING, dp
    assert du <= TOL_PU + FIXTURE_ROUNDING, du
    return ds, dp, du


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_full_run_matches_oracle(name):
    fx = load(name)
    c = configs.build(name)
    assert c.split.te == int(fx["split_te"][0])
    r = api.Simulator(c.problem).run(c.split, c.s0(), c.inflow_sat)
    check_record(r, fx)
    ds, dp, du = check_fields(r, fx)
    print(f"{name}: {r.record.te} steps, {r.record.tm_total} rebuilds, max|ds| {ds:.2e}, p {dp:.2e}, u {du:.2e}")


def check_fields_vs_truth(run, fx, prefix=""):
    """C3's channelised field (K spans 1.6e7, cond(M) ~ 2e9) puts the exact
    answer ~2e-7 (relative L2 in u) away from ANY double-precision direct
    solve, the oracle's included (tools/make_fixtures.py measures it against
    the oracle compiled with long double). Each field must match the oracle to
    the 1e-8 bar, or, where the oracle's own double-precision error exceeds
    that bar, be at least as close to the extended-precision answer as the
    oracle is (factor 3 for solver-dependent roundoff constants)."""
    out = {}
    for nm in ("s", "p", "u"):
        g, o, x = getattr(run, nm + "_final"), fx[prefix + nm], fx[prefix + "ld_" + nm]
        if nm == "s":
            d_go, d_gx, d_ox = (float(np.max(np.abs(a - b))) for a, b in ((g, o), (g, x), (o, x)))
        else:
            d_go, d_gx, d_ox = rel_l2(g, o), rel_l2(g, x), rel_l2(o, x)
        ok = d_go <= 1e-8 + FIXTURE_ROUNDING or d_gx <= max(1e-8, 3.0 * d_ox) + FIXTURE_ROUNDING
        assert ok, (nm, {"gpu_vs_oracle": d_go, "gpu_vs_exact": d_gx, "oracle_vs_exact": d_ox})
        out[nm] = {"gpu_vs_oracle": d_go, "gpu_vs_exact": d_gx, "oracle_vs_exact": d_ox}
    return out


def test_c3_two_pass_to_breakthrough_plus_50():
    """C3 as BASELINE states it: run to water breakthrough, then to
    breakthrough + 50 %. The GPU must break through at the oracle's step
    (5,501), make the oracle's decisions at every step of both passes and
    match its fields (see check_fields_vs_truth for the accuracy yardstick)."""
    fx = load("C3")
    c = configs.build("C3")
    sim = api.Simulator(c.problem)
    r1 = sim.run(c.split, c.s0(), c.inflow_sat)
    assert r1.record.breakthrough_step == int(fx["pass1_meta_int"][3])
    check_record(r1, fx, "pass1_", exact_yardstick=True)
    e1 = check_fields_vs_truth(r1, fx, "pass1_")
    te2 = configs.breakthrough_plus_50(r1.record.breakthrough_step)
    assert te2 == int(fx["split_te"][0])
    sp2 = dataclasses.replace(c.split, stop_on_breakthrough=False, te=te2)
    r2 = sim.run(sp2, c.s0(), c.inflow_sat)
    check_record(r2, fx, exact_yardstick=True)
    e2 = check_fields_vs_truth(r2, fx)
    print(f"C3: breakthrough {r1.record.breakthrough_step}, te {te2}; pass 1 {e1}; pass 2 {e2}")


def _sketch_rel_err(x, fx, nm):
    """Estimate |x - x_ref| / |x_ref| from the stored Rademacher sketch
    (E[(r.d)^2] = |d|^2 for r with independent +-1 entries)."""
    from golden_io import rademacher
    sk = np.array([rademacher(x.size, k) @ x for k in range(fx[nm + "_sketch"].size)])
    d = sk - fx[nm + "_sketch"]
    return float(np.sqrt(np.mean(d * d)) / fx[nm + "_norm"][0])


def check_sketched_vs_truth(r, fx, fl, prefix=""):
    """C5-size fields: s at every cell, p and u through the sketch and the
    1/256 subsample, against the oracle fixture fx; where fl (the
    extended-precision run, keys prefixed `prefix`) exists, a field may instead
    be at least as close to it as the double-precision oracle is (factor 3),
    the rule of check_fields_vs_truth."""
    from golden_io import subsample_idx

    def dense_s(f, pre=""):
        s = np.zeros(r.s_final.size)
        s[f[pre + "s_nz_idx"]] = f[pre + "s_nz_val"]
        return s
    s_o = dense_s(fx)
    errs = {"s": {"gpu_vs_oracle": float(np.max(np.abs(r.s_final - s_o)))}}
    if fl is not None:
        s_x = dense_s(fl, prefix)
        errs["s"]["gpu_vs_exact"] = float(np.max(np.abs(r.s_final - s_x)))
        errs["s"]["oracle_vs_exact"] = float(np.max(np.abs(s_o - s_x)))
    for nm, x in (("p", r.p_final), ("u", r.u_final)):
        e = {"gpu_vs_oracle": _sketch_rel_err(x, fx, nm)}
        idx = subsample_idx(x.size)
        e["gpu_vs_oracle_sub"] = rel_l2(x[idx], fx[nm + "_sub"])
        if fl is not None:
            e["gpu_vs_exact"] = _sketch_rel_err(x, fl, prefix + nm)
            d = fx[nm + "_sketch"] - fl[prefix + nm + "_sketch"]
            e["oracle_vs_exact"] = float(np.sqrt(np.mean(d * d)) / fl[prefix + nm + "_norm"][0])
        errs[nm] = e
    for nm, e in errs.items():
        tol = TOL_S if nm == "s" else TOL_PU
        strict = e["gpu_vs_oracle"] <= tol and e.get("gpu_vs_oracle_sub", 0.0) <= tol
        yard = "gpu_vs_exact" in e and e["gpu_vs_exact"] <= max(tol, 3.0 * e["oracle_vs_exact"])
        assert strict or yard, (nm, e)
    return errs


def test_c5_full_run_matches_oracle():
    """C5 (16.8 M cells, 16,384 subdomains, interface dim 65,024): the whole
    500-step run vs the oracle (banded interface LU): decisions and counters
    exact; s at every cell, p and u through the sketch and a 1/256 subsample.
    Where the oracle's own double-precision answer is farther than 1e-8 from
    the extended-precision one (run_C5_ld.npz), the GPU must be at least as
    close to the latter (the C3 rule, check_fields_vs_truth)."""
    fx = load("C5")
    ld_path = os.path.join(GOLDEN, "run_C5_ld.npz")
    fl = dict(np.load(ld_path)) if os.path.exists(ld_path) else None
    c = configs.build("C5")
    assert c.split.te == int(fx["split_te"][0])
    r = api.Simulator(c.problem).run(c.split, c.s0(), c.inflow_sat)
    check_record(r, fx)
    assert r.record.tm_total >= 6  # the initial MRCM solve plus >= 5 rebuilds

    errs = check_sketched_vs_truth(r, fx, fl)
    print(f"C5: rebuilds at {r.record.update_steps}, errors {errs}")
