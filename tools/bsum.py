"""Print the headline, branch split and top kernels of bench JSON lines
(developer tool). Usage: python tools/bsum.py FILE... [--top N]"""
import json
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
for f in args:
    if f.isdigit():
        continue
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    roof = d.get("roofline") or {}
    print(f"{f}: value {d['value']:.1f} {d['unit']} ms/step {d.get('ms_per_step', 0):.4f} "
          f"rebuilds {d.get('rebuilds_in_timed_steps')} launches {d.get('gpu_launches')} "
          f"roofline {roof.get('kernel')} frac {roof.get('frac')}")
    for nm, b in (d.get("branch_split") or {}).items():
        print(f"    {nm:14s} {b['steps']:5d} steps  {b['ms_per_step']:.4f} ms")
    for k, v in list((d.get("kernels") or {}).items())[:top]:
        print(f"    {k:22s} {v['launches']:6d} share {v['share']:.3f} avg {v['avg_us']:9.2f} us  {v.get('achieved', '')}")
