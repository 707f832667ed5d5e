"""Summarise an ncu launch list (developer tool).

Input: the CSV written by
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file X.csv <cmd>
Output: per-kernel launches, total, average and share (cold-cache and
serialised per launch: compare shares, not absolutes).
Usage: python tools/launch_list.py X.csv [title]
"""
import csv
import re
import sys


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = None
    agg = {}
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[hdr["Kernel Name"]]
        name = re.sub(r"\(.*", "", name).replace("mpm2p::", "").replace("(anonymous namespace)::", "")
        unit = r[hdr["Metric Unit"]]
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        u = unit.strip().lower()
        us = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {title}")
    print("# per-launch times are cold-cache and serialised: compare SHARES, not absolutes")
    print(f"# launches: {n}  total: {tot / 1e3:.3f} ms")
    print(f"{'kernel':44s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>9s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:44]:44s} {c:8d} {t / 1e3:10.3f} {t / c:9.2f} {100 * t / tot:6.2f}%")


if __name__ == "__main__":
    main()
