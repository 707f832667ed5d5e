"""Warp-stall samples of one kernel aggregated by CUDA source line (developer
tool; needs -lineinfo and an ncu report captured with --import-source on).
Usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern, "--launch-count", "1"], capture_output=True, text=True).stdout
fname = "?"
rows = []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0].isdigit():
        try:
            rows.append((fname, int(r[0]), r[1].strip(), float(r[4]), float(r[7] or 0)))
        except ValueError:
            pass
tot = sum(x[3] for x in rows) or 1.0
print(f"samples {tot:.0f}")
for f, ln, src, s, ex in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5d} inst {ex:12.0f}  {src[:90]}")
