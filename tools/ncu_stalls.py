"""Stall breakdown of one kernel from an ncu report's SASS source page
(developer tool): totals per stall reason and the hottest instructions.
Usage: python tools/ncu_stalls.py REPORT KERNEL_REGEX [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: sum(f(r[ix[k]]) for r in data) for k in reasons}
allm = sum(f(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data)
print(f"samples {allm:.0f}")
for k, v in sorted(tot.items(), key=lambda t: -t[1])[:10]:
    print(f"  {k:24s} {v:8.0f}  {100 * v / max(allm, 1):5.1f}%")
# instruction-class totals
cls = {}
for r in data:
    op = r[ix["Source"]].split()
    op = [t for t in op if not t.startswith("@")]
    name = op[0].split(".")[0] if op else "?"
    cls.setdefault(name, [0, 0])
    cls[name][0] += f(r[ix["Warp Stall Sampling (All Samples)"]])
    cls[name][1] += f(r[ix["Instructions Executed"]])
print("by opcode (samples, executed):")
for k, v in sorted(cls.items(), key=lambda t: -t[1][0])[:14]:
    print(f"  {k:10s} {v[0]:8.0f} {v[1]:10.0f}")
print("hottest:")
for r in sorted(data, key=lambda r: -f(r[ix["Warp Stall Sampling (All Samples)"]]))[:top]:
    st = sorted(((f(r[ix[k]]), k[6:]) for k in reasons), reverse=True)[:2]
    print(f"  {r[ix['Address']][-5:]} {f(r[ix['Warp Stall Sampling (All Samples)']]):6.0f} {r[ix['Source']].strip()[:60]:60s} "
          + " ".join(f"{k}={v:.0f}" for v, k in st))
