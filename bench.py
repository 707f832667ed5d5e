#!/usr/bin/env python3
"""Benchmark of the MPM-2P velocity-update + saturation-update path on B200.

A "step" is one Algorithm-1 iteration of the reference driver
(proj/src/simulation.cpp:262-329): CFL reduction, `cn` explicit upwind
saturation substeps, conductivity + drift test, and one velocity update
(MPM-2P reuse, or a full MRCM rebuild when the device-side drift test says
so). The headline workload is C5, the largest single-GPU config of
BASELINE.json (4096^2 cells, 128x128 subdomains of 32x32, interface dim
65,024); C2 (configs[1]) is measured in the same run as a second workload
under "also". Inputs are seeded synthetic fields (no dataset).

  value    velocity updates/s over the timed steps, inputs resident in HBM;
           device time of each step's CUDA-graph replay from CUDA events on
           the library's stream (timer slots 14/15 around cudaGraphLaunch, so
           host-side driver work and first-use graph capture are excluded),
           L2 flushed before every step; split by branch (MPM-2P / MRCM)
  e2e      the same metric for whole simulations through the C ABI with host
           buffers (context creation + mpm2p_run incl. all H2D/D2H copies;
           C3: both passes, to breakthrough and to breakthrough + 50 %)
  cpu_baseline / --impl reference
           the CPU restatement of the reference (oracle/, C++ -O3, 1 thread:
           the reference has no threads) on a bounded sample of the same run
           (C5: the banded interface LU — the reference's dense LU would need
           34 GB); CPU model and nproc recorded

Multi-GPU (torchrun): N independent replicas, one per GPU, no data-path
collective (the sharded path is future work); value is the
sum over ranks divided by the max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPM-2P velocity updates/s + FV cell-updates/s (fp64) at 1 B200; % HBM roofline"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        return ws, rank, local, dist, torch
    return ws, rank, local, None, None


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


FP64_PEAK_TFLOPS = 34.2  # measured DFMA peak on this pool (profiles/fp64_peaks_r01.log)


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# kernels launched on the side stream (split downscale: the kappa_n operator is
# factored concurrently with the particular / interface chain) — timed, but
# not on the step's critical path, so never picked as the roofline kernel
SIDE_STREAM = ("k_ds_band", "k_ds_factor")


def kernel_work(name, cfg, sz, dim):
    """Algorithmic bytes / flops per launch of each kernel."""
    cells, faces = sz.cells, sz.faces
    n, B, ns = sz.sub_nx * sz.sub_ny, sz.sub_nx, sz.n_sub
    table = {
        "k_upwind": ("hbm", 32.0 * cells),                       # s r/w + 2 faces of u
        "k_cfl": ("hbm", 16.0 * cells),
        # the driver's per-step launch reads s, K, kappa_m and writes kappa and the
        # fused transmissibilities T (2 faces per cell): 24 + 8 + 16 B per cell
        "k_kappa": ("hbm", 48.0 * cells),
        "k_part_solve": ("hbm", ns * n * (16.0 * B + 24.0)),     # Lcol, Lrow, D, x r/w
        "k_ds_solve": ("fp64", ns * (n * B * B + 4.0 * n * B)),  # banded LDL^T factor + 2 sweeps
        # blocked DMMA downscale (band_blk.cuh): factor + forward sweep; backward sweep from the stored panels
        "k_ds_blk_factor": ("fp64", ns * (n * B * B + 2.0 * n * B)),
        "k_ds_blk_solve": ("hbm", ns * n * (8.0 * B + 8.0 + 16.0)),  # X panels + t1 read, x written, p written
        "k_ds_factor": ("fp64", ns * n * B * B),                # split downscale: factor (side stream)
        "k_ds_sweep": ("hbm", ns * n * (16.0 * B + 24.0)),       # split downscale: 2 sweeps with the stored factor
        "k_factor_solve": ("fp64", ns * (n * B * B + 4.0 * n * B * (1 + sz.nhat / max(ns, 1)))),
        "k_gemv": ("hbm", 8.0 * dim * dim),
        # MPM-2P right-hand side: p^m, two faces of T(kappa_n), q read; X written; per subdomain edge
        # kappa_n and the static pressure drop read, WU written, WU / ET read back: 40 B
        "k_mpm_rhs": ("hbm", 40.0 * cells + 40.0 * ns * sz.sub_nx * 4),
        # MPM-2P recombination: per subdomain edge PU, WU and the max_hom homogeneous traces read, RU written
        "k_recon_mpm": ("hbm", 8.0 * ns * sz.sub_nx * 4 * (3.0 + sz.nhat / max(ns, 1))),
        # velocity scatter: X (downscaled potential), two faces of T, q read; two faces of u written
        "k_ds_u_div": ("hbm", 48.0 * cells),
        "k_ds_prep": ("hbm", 72.0 * cells),
        # downscale rhs alone (operator formed by the factor): q read, X written; edges: RU/skel in, EU/ET out
        "k_ds_rhs": ("hbm", 16.0 * cells + 40.0 * ns * sz.sub_nx * 4),
        "k_ds_u": ("hbm", 32.0 * faces),
        "k_divres": ("hbm", 24.0 * cells + 8.0 * faces),
        "k_trans": ("hbm", 16.0 * cells + 8.0 * faces),
    }
    if name == "k_cr_gemv" and dim > 16384:
        # interface solve by block cyclic reduction (blocktri.cu): nb block rows (one per subdomain
        # row) padded to S. Per level with e eliminated blocks three launches: c_o = D_o^-1 y_o (e
        # blocks read), y_e -= Lo_e c + Up_e c (2e), backward x_o = c_o - P_o x - Q_o x (2e); the
        # top solve reads one block. The per-launch figure is the solve's bytes over its launches
        # (22 at nb = 128)
        nb = max(1, round(ns ** 0.5))  # subdomain rows (the configs' decompositions above dim 16,384 are square)
        S = -(-(dim // nb) // 64) * 64
        blocks, launches, lv = 1, 1, nb
        while lv > 1:
            blocks += 5 * (lv // 2)
            launches += 3
            lv -= lv // 2
        return ("hbm", 8.0 * S * S * blocks / launches)
    return table.get(name)


def run_ours(args, ws, rank, local, dist, torch, config=None, steps=None):
    import ctypes
    import dataclasses
    os.environ["MPM2P_GRAPH_TIMING"] = "1"  # replay-only device timing (read at context creation)
    from paper_2103_11050_b200 import api, configs
    lib = api.product_lib()
    if ws > 1:
        lib.set_device(local)
    cfg = configs.build(config or args.config)
    n_steps = steps if steps is not None else args.steps
    te_needed = args.warmup + n_steps + 1
    split = cfg.split
    if cfg.two_pass or (split.te and split.te < te_needed + args.profile_steps):
        # room for the timed and the profiled window (the e2e run keeps the config's own schedule)
        split = dataclasses.replace(split, te=max(te_needed + args.profile_steps, split.te or 0),
                                    stop_on_breakthrough=False)
    sim = api.Simulator(cfg.problem, lib)
    sz = sim.sizes
    dim = sim.dim
    cn = split.cn
    sim.run_begin(split, cfg.s0(), cfg.inflow_sat)
    for _ in range(args.warmup):
        if sim.run_step() is None:
            break
    sampler = ClockSampler(local)
    if ws > 1:
        dist.barrier()
        torch.cuda.synchronize()
    sampler.start()
    dev_ms = 0.0
    span_ms = 0.0
    done = 0
    branch = {0: [], 1: []}
    launches0 = _launches(sim)
    t_wall0 = time.perf_counter()
    ms = ctypes.c_double()
    for _ in range(n_steps):
        lib.flush_l2(sim.h)
        lib.timer_record(sim.h, 0)
        rec = sim.run_step()
        lib.timer_record(sim.h, 1)
        if rec is None:
            break
        lib.timer_elapsed(sim.h, 14, 15, ctypes.byref(ms))  # the graph replay alone
        dev_ms += ms.value
        branch[rec["rebuilt"]].append(ms.value)
        lib.timer_elapsed(sim.h, 0, 1, ctypes.byref(ms))    # stream span incl. host-side driver work
        span_ms += ms.value
        done += 1
    wall = time.perf_counter() - t_wall0
    launches = _launches(sim) - launches0
    clocks = sampler.stop()
    if ws > 1:
        dev_ms_max, done_total = reduce_over_ranks(dev_ms, done, dist, "cuda")
    else:
        dev_ms_max, done_total = dev_ms, float(done)
    # per-kernel device times over a separate profiled window (same stream, CUDA events)
    prof = _profile(sim, lib, min(args.profile_steps, max(0, split.te - 1 - args.warmup - done)))
    sim.run_end()
    sim.close()
    # end-to-end: whole simulations through the C ABI with host buffers
    e2e = None
    if not args.skip_e2e:
        e2e = _e2e(api, lib, cfg, args)
    split_out = {}
    for b, nm in ((0, "mpm2p"), (1, "mrcm_rebuild")):
        v = branch[b]
        if v:
            split_out[nm] = {"steps": len(v), "ms_per_step": sum(v) / len(v),
                             "updates_per_s": len(v) / (sum(v) / 1e3)}
    return dict(cfg=cfg, split=split, sz=sz, dim=dim, cn=cn, done=done, done_total=done_total,
                dev_ms=dev_ms, dev_ms_max=dev_ms_max, span_ms=span_ms, wall=wall, rebuilds=len(branch[1]),
                clocks=clocks, launches=launches, prof=prof, e2e=e2e, branch_split=split_out)


def reduce_over_ranks(dev_ms, done, dist, device):
    """Max over ranks of the device time, sum over ranks of the work done."""
    import torch
    t = torch.tensor([float(dev_ms)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(done)], device=device, dtype=torch.float64)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), float(n.item())


def _launches(sim):
    import ctypes
    buf = ctypes.create_string_buffer(1 << 16)
    sim.lib.profile_report(sim.h, buf, len(buf))
    for line in buf.value.decode().splitlines():
        p = line.split()
        if p and p[0] == "__launches__":
            return int(p[1])
    return 0


def _profile(sim, lib, steps):
    import ctypes
    if steps <= 0:
        return {}
    lib.profile_enable(sim.h, 1)
    n = 0
    for _ in range(steps):
        if sim.run_step() is None:
            break
        n += 1
    buf = ctypes.create_string_buffer(1 << 16)
    lib.profile_report(sim.h, buf, len(buf))
    lib.profile_enable(sim.h, 0)
    out = {}
    for line in buf.value.decode().splitlines():
        p = line.split()
        if len(p) == 3 and p[0] != "__launches__":
            out[p[0]] = {"launches": int(p[1]), "total_ms": float(p[2])}
    out["__steps__"] = n
    return out


def _simulate(api, lib, cfg):
    """One whole simulation through the C ABI: create + run (+ C3's second pass).
    Returns (steps, rebuilds, seconds); the context teardown after the run is
    not in the timed region."""
    import dataclasses
    t0 = time.perf_counter()
    sim = api.Simulator(cfg.problem, lib)
    try:
        res = sim.run(cfg.split, cfg.s0(), cfg.inflow_sat)
        steps, rebuilds = res.record.te - 1, res.record.tm_total
        if cfg.two_pass:  # "until breakthrough + 50 %": second pass with te from the first
            from paper_2103_11050_b200 import configs
            b = res.record.breakthrough_step
            if b < 0:
                raise RuntimeError(f"{cfg.name}: no breakthrough in pass 1")
            sp2 = dataclasses.replace(cfg.split, stop_on_breakthrough=False, te=configs.breakthrough_plus_50(b))
            res2 = sim.run(sp2, cfg.s0(), cfg.inflow_sat)
            steps += res2.record.te - 1
            rebuilds += res2.record.tm_total
        return steps, rebuilds, time.perf_counter() - t0
    finally:
        sim.close()


def _e2e(api, lib, cfg, args, reps=3):
    """Whole simulations through the C ABI with host buffers: context creation
    (uploads K, q, the boundary spec; static operators) + mpm2p_run (s0 upload,
    every Algorithm-1 step with its scalar readback, final s/p/u download).
    Teardown is outside the timed region (cudaFree timing is noisy). Median of
    `reps` runs after one untimed run; all samples are reported."""
    walls = []
    # one untimed simulation first: process-level one-time costs (module
    # loading, allocator pools) are not per-simulation work; short runs
    # (< 1 s) take the median of five
    if _simulate(api, lib, cfg)[2] < 1.0:
        reps = max(reps, 5)
    for _ in range(reps):
        steps, rebuilds, w = _simulate(api, lib, cfg)
        walls.append(w)
    wall = sorted(walls)[len(walls) // 2]
    cells = cfg.cells
    faces = (cfg.problem.nx + 1) * cfg.problem.ny + cfg.problem.nx * (cfg.problem.ny + 1)
    nb = 2 * (cfg.problem.nx + cfg.problem.ny)
    passes = 2 if cfg.two_pass else 1
    h2d = passes * (8 * cells * 2 + 12 * nb)  # K + s0 + boundary spec
    d2h = passes * 8 * (2 * cells + faces) + 256 * (steps + passes)  # final s, p, u + per-step scalars
    return {"value": steps / wall, "unit": "velocity_updates/s", "h2d_bytes_per_step": h2d / max(steps, 1),
            "d2h_bytes_per_step": d2h / max(steps, 1), "wall_s_per_simulation": wall, "steps": steps,
            "rebuilds": rebuilds, "passes": passes, "wall_samples_s": [round(w, 4) for w in walls]}


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def cpu_reference(cfg, split, budget_s, threads=1):
    """The reference's CPU path (oracle restatement, C++ -O3) on a bounded
    sample: the initial MRCM solve (reported, not in the rate), then as many
    Algorithm-1 steps of the same run as fit in budget_s. threads = 1 is the
    reference as it is (it has no threads); threads > 1 runs the port's
    per-subdomain loops on that many cores (same results bit for bit)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import oracle_lib
    from paper_2103_11050_b200 import api
    lib = oracle_lib()
    lib.dll.oracle_set_threads(int(threads))
    sim = api.Simulator(cfg.problem, lib)
    t0 = time.perf_counter()
    sim.run_begin(split, cfg.s0(), cfg.inflow_sat)
    t_begin = time.perf_counter() - t0
    n = 0
    br = {0: [], 1: []}
    t1 = time.perf_counter()
    while time.perf_counter() - t1 < budget_s:
        ts = time.perf_counter()
        r = sim.run_step()
        if r is None:
            break
        br[r["rebuilt"]].append(time.perf_counter() - ts)
        n += 1
    el = time.perf_counter() - t1
    sim.run_end()
    sim.close()
    iface = "banded partial-pivot LU of the interface matrix (dense LU: 34 GB)" if cfg.name == "C5" else \
        "dense partial-pivot LU of the interface matrix, as the reference"
    lib.dll.oracle_set_threads(1)
    how = "single thread (the reference is single-threaded and cannot be built here: no Eigen)" if threads == 1 else \
        f"{threads} threads over the per-subdomain loops (the port's own; the reference has none)"
    return {"value": n / el if el > 0 else 0.0, "unit": "velocity_updates/s", "cores": int(threads), "kind": "port",
            "sample": f"{cfg.name}: initial MRCM solve ({t_begin:.2f} s, not in the rate) then the first {n} "
                      f"Algorithm-1 steps ({el:.1f} s, {len(br[1])} rebuilds) of the same run; oracle/ C++ -O3 "
                      f"{how}; {iface}",
            "branch_s_per_step": {"mpm2p": (sum(br[0]) / len(br[0])) if br[0] else None,
                                  "mrcm_rebuild": (sum(br[1]) / len(br[1])) if br[1] else None},
            "initial_solve_s": t_begin, "cpu": cpu_info(), "steps": n, "seconds": el}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--also", default="C2", help="further workloads measured in the same run (N=1 only)")
    ap.add_argument("--also-steps", type=int, default=300)
    ap.add_argument("--also-cpu-budget", type=float, default=10.0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local, dist, torch = _dist()
    from paper_2103_11050_b200 import configs

    if args.impl == "reference":
        if rank != 0:
            return
        cfg = configs.build(args.config)
        import dataclasses
        split = dataclasses.replace(cfg.split, stop_on_breakthrough=False,
                                    te=max(cfg.split.te or 0, args.warmup + args.steps + 1))
        cb = cpu_reference(cfg, split, args.cpu_budget)
        # for information: the same sample with the port's per-subdomain loops on every host core
        # (the reference has no threads, so the line's value stays the single-thread figure)
        ca = cpu_reference(cfg, split, args.cpu_budget, threads=os.cpu_count() or 1)
        line = {"metric": METRIC, "value": cb["value"], "unit": "velocity_updates/s", "impl": "reference",
                "n_gpus": ws, "steps": cb["steps"], "warmup": 0, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded field generator)",
                "config": {"workload": cfg.name, "description": cfg.description},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "port_all_cores": {k: ca[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": "velocity_updates/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    r = run_ours(args, ws, rank, local, dist, torch)
    also = {}
    if args.also and ws == 1:
        for name in [x for x in args.also.split(",") if x and x.upper() != r["cfg"].name]:
            ra = run_ours(args, ws, rank, local, dist, torch, config=name, steps=args.also_steps)
            la = build_line(ra, args, ws, cpu_budget=args.also_cpu_budget)
            also[ra["cfg"].name] = {k: la[k] for k in ("value", "unit", "ms_per_step", "steps", "cell_updates_per_s",
                                                       "branch_split", "roofline", "e2e", "cpu_baseline",
                                                       "gpu_launches", "config", "clocks")}
    if rank != 0:
        if dist is not None:
            dist.barrier()
        return
    line = build_line(r, args, ws, cpu_budget=args.cpu_budget)
    if also:
        line["also"] = also
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()


def build_line(r, args, ws, cpu_budget):
    cfg, sz, dim = r["cfg"], r["sz"], r["dim"]
    secs = r["dev_ms_max"] / 1e3
    value = r["done_total"] / secs
    cells = sz.cells
    cell_updates = r["done_total"] * r["cn"] * cells / secs
    hbm_peak, peak_src = _peaks()
    # roofline of the dominant kernel (largest share of profiled device time)
    prof = r["prof"]
    kern = {k: v for k, v in prof.items() if not k.startswith("__")}
    roof = None
    shares = {}
    tot = sum(v["total_ms"] for v in kern.values()) or 1.0
    for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["total_ms"]):
        shares[k] = {"share": round(v["total_ms"] / tot, 4), "launches": v["launches"],
                     "avg_us": round(1e3 * v["total_ms"] / v["launches"], 3)}
        if k in SIDE_STREAM:
            shares[k]["stream"] = "side (concurrent with the critical path)"
        w = kernel_work(k, cfg, sz, dim)
        if w:
            avg_s = v["total_ms"] / v["launches"] / 1e3
            if w[0] == "hbm":
                ach = w[1] / avg_s / 1e9
                shares[k]["achieved"] = f"{ach:.1f} GB/s ({ach / hbm_peak:.3f} of HBM)"
            else:
                ach = w[1] / avg_s / 1e12
                shares[k]["achieved"] = f"{ach:.3f} TFLOP/s ({ach / FP64_PEAK_TFLOPS:.3f} of fp64 DFMA)"
    for k in sorted(kern, key=lambda k: -kern[k]["total_ms"]):
        w = kernel_work(k, cfg, sz, dim)
        if not w or k in SIDE_STREAM:
            continue
        v = kern[k]
        avg_s = v["total_ms"] / v["launches"] / 1e3
        if w[0] == "hbm":
            ach = w[1] / avg_s / 1e9
            roof = {"kernel": k, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ach / hbm_peak, "traffic": None, "peak_source": peak_src,
                    "algorithmic_per_launch": w[1], "avg_launch_us": avg_s * 1e6}
        else:
            ach = w[1] / avg_s / 1e12
            roof = {"kernel": k, "bound": "fp64", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP64_PEAK_TFLOPS, "traffic": None,
                    "peak_source": "measured DFMA peak (profiles/fp64_peaks_r01.log)",
                    "algorithmic_per_launch": w[1], "avg_launch_us": avg_s * 1e6}
        break
    if roof is not None:  # dram bytes per launch from the committed ncu --set full capture
        tpath = None
        for rnd in ("r02", "r01"):  # the latest round's capture
            cand = os.path.join(ROOT, "profiles", f"ncu_traffic_{rnd}_{cfg.name}.json")
            if os.path.exists(cand):
                tpath = cand
                break
        try:
            with open(tpath or "") as f:
                tr = {k.split("::")[-1]: v for k, v in json.load(f).items()}
            # keys carry template arguments (k_ds_solve_r<16>): match the launcher name as a prefix
            hit = [v for k, v in tr.items() if k == roof["kernel"] or k.startswith(roof["kernel"] + "_r<")
                   or k.startswith(roof["kernel"] + "_t<") or k.startswith(roof["kernel"] + "<")
                   or k.startswith(roof["kernel"] + "_tile")]
            roof["traffic"] = hit[0] if hit else None
            roof["traffic_source"] = f"{os.path.relpath(tpath, ROOT)} (ncu dram__bytes_read+write per launch)"
        except (OSError, ValueError):
            pass
    cpu = None
    if not args.skip_cpu and ws == 1 and cpu_budget > 0:
        import dataclasses
        cpu_split = dataclasses.replace(r["split"], stop_on_breakthrough=False)
        cb = cpu_reference(cfg, cpu_split, cpu_budget)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "branch_s_per_step",
                                  "initial_solve_s", "cpu")}
    return {
        "metric": METRIC, "value": value, "unit": "velocity_updates/s", "n_gpus": ws, "steps": r["done"],
        "warmup": args.warmup, "ms_per_step": r["dev_ms_max"] / max(r["done"], 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded field generator)",
        "config": {"workload": cfg.name, "description": cfg.description, "cells": cells,
                   "subdomains": sz.n_sub, "interface_dim": dim, "cn": r["cn"],
                   "l2": "flushed before every timed step",
                   "timing": "CUDA events around each step's graph replay (host driver work excluded; "
                             "stream_ms_per_step includes it)",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
        "cell_updates_per_s": cell_updates,
        "branch_split": r["branch_split"],
        "rebuilds_in_timed_steps": r["rebuilds"],
        "stream_ms_per_step": r["span_ms"] / max(r["done"], 1),
        "host_wall_ms_per_step": 1e3 * r["wall"] / max(r["done"], 1),
        "gpu_launches": r["launches"],
        "roofline": roof,
        "kernels": shares,
        "clocks": r["clocks"],
        "e2e": r["e2e"],
        "cpu_baseline": cpu,
    }


if __name__ == "__main__":
    main()
