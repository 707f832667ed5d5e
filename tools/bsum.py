"""Print the headline and the top kernels of bench JSON lines (developer tool)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    print(f"{f}: value {d['value']:.1f} {d['unit']} ms/step {d['ms_per_step']:.4f} rebuilds {d.get('rebuilds_in_timed_steps')}"
          f" roofline {d.get('roofline', {}).get('kernel')} frac {d.get('roofline', {}).get('frac')}")
    for k, v in list((d.get("kernels") or {}).items())[:8]:
        print(f"    {k:18s} share {v['share']:.3f} avg {v['avg_us']:9.1f} us  {v.get('achieved', '')}")
