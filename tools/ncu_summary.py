"""Per-kernel summary of an `ncu --set full` report (developer tool).

Writes, per kernel (averaged over its captured launches): duration, DRAM
read+write bytes, SM / DRAM throughput, FP64 pipe activity, registers,
achieved occupancy and the top warp-stall reasons; optionally the per-launch
DRAM traffic JSON that bench.py reads for roofline.traffic.
Usage: python tools/ncu_summary.py REPORT [--traffic-json OUT.json] > summary.txt
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__grid_size",
]


def to_bytes(v, unit):
    u = unit.strip().lower()
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)


def main():
    rep = sys.argv[1]
    out_json = None
    if "--traffic-json" in sys.argv:
        out_json = sys.argv[sys.argv.index("--traffic-json") + 1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    agg = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").split("::")[-1]
        a = agg.setdefault(name, {"n": 0})
        a["n"] += 1
        for m in METRICS:
            if m not in d or d[m] in ("", "n/a"):
                continue
            if m.startswith("dram__bytes"):
                v = to_bytes(d[m], u[m])
            elif m == "gpu__time_duration.sum":
                v = float(d[m].replace(",", "")) * (1e-3 if u[m].strip() == "ns" else (1e3 if u[m].strip() == "ms" else 1))
            else:
                v = float(d[m].replace(",", ""))
            a[m] = a.get(m, 0.0) + v
    traffic = {}
    print(f"# ncu --set full summary of {rep} (cold cache, serialised; per-launch averages)")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
        n = a["n"]
        g = lambda m: a.get(m, 0.0) / n  # noqa: E731
        tr = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
        traffic[name] = tr
        print(f"{name}  (launches captured: {n})")
        print(f"   duration {g('gpu__time_duration.sum'):.2f} us   grid {g('launch__grid_size'):.0f}   "
              f"regs {g('launch__registers_per_thread'):.0f}   warps active {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%")
        print(f"   DRAM read+write {tr / 1e6:.3f} MB   DRAM thrpt {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}%   "
              f"SM thrpt {g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f}%   FP64 pipe {g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%")
        print(f"   inst executed {g('smsp__inst_executed.sum'):.0f}")
    if out_json:
        with open(out_json, "w") as f:
            json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main()
