"""Print value / ms per step and the top kernels of a bench JSON line (developer tool)."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["value"], 2), round(d["ms_per_step"], 4), "launches", d.get("gpu_launches"))
    for n, v in list(d.get("kernels", {}).items())[:16]:
        print(f"   {n:22s} {v['launches']:6d} {v['avg_us']:9.2f} {v['share']:.3f} {v.get('achieved', '')}")
