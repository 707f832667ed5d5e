"""Summarise an ncu report: per-kernel key metrics and the hottest SASS lines."""
import csv, io, subprocess, sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None

def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

mets = ("gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,"
        "dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,"
        "launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,"
        "smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,"
        "smsp__average_warp_latency_per_inst_issued.ratio,lts__t_bytes.sum")
rows = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv", "--metrics", mets]))))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:60])
    for m in mets.split(","):
        print(f"   {m:70s} {d.get(m, '')}")
if kern:
    src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "-k", kern, "--launch-count", "1"]))))
    hh = src[1]
    idx = {k: j for j, k in enumerate(hh)}
    def f(x):
        try: return float(x)
        except: return 0.0
    data = [r for r in src[2:] if len(r) == len(hh) and r[0].startswith("0x")]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(f(r[idx[key]]) for r in data) or 1
    print("hot SASS (%):")
    for j, r in enumerate(data):
        v = f(r[idx[key]])
        if v / tot > 0.01:
            print(f"  {j:5d} {100*v/tot:5.1f}%  {r[1][:80]}")
