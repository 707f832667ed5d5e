import sys, dataclasses
sys.path.insert(0, "/root/repo")
from paper_2103_11050_b200 import api, configs
for name in ["C1", "C2", "C3", "C4"]:
    c = configs.build(name, te_override=60)
    r = api.Simulator(c.problem).run(c.split, c.s0())
    print(name, "min_rcond", r.record.min_rcond, "rebuilds", r.record.tm_total)
