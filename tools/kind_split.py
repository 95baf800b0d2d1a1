"""C5 kernel times per scene family: 4096 scenes of one kind each (device-resident inputs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_17340_b200 import Planner
from paper_2509_17340_b200.workloads import plan_config, scenes, KIND_NAMES

cfg = plan_config()
for kind in (1, 2, 3):
    d = scenes(4096, kinds=kind)
    p = Planner(cfg, max_scenes=4096, max_points=int(d["offsets"][-1]) + 1, profile=True)
    for i in range(3):
        p.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"] + np.uint64(i), d["seeds"])
    p.kernel_times_reset()
    for i in range(3):
        p.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"] + np.uint64(10 + i), d["seeds"])
    kt = p.kernel_times()
    print(KIND_NAMES[kind], {k: round(v[0] / 3, 3) for k, v in kt.items() if v[0] / 3 > 0.05})
    p.close()
