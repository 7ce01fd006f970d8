import os, sys, json
sys.path.insert(0, os.getcwd())
import bench, torch
from paper_2511_11581_b200 import pattn
from workloads import CONFIGS
pattn.load()
dev = torch.device("cuda", 0)
for name in ("c3_mixed8b", "c2_decode8b"):
    case = bench.Case(CONFIGS[name], 3003, dev, pattn, 2, 0, 126 << 20)
    for rep in range(3):
        a, _ = bench.timed(case, 100, 10, lambda: None, with_events=False)
        b, _ = bench.timed(case, 100, 10, lambda: None, with_events=True)
        print(name, "no events %.2f us" % (a * 1e3), "with events %.2f us" % (b * 1e3))
