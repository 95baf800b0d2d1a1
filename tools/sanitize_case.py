"""Small workloads for compute-sanitizer (racecheck / memcheck / synccheck):
one C1 plan cycle through the single-scene C ABI (latency kernels) and one
160-scene batch through amppi_cycle_batch (fused per-scene snapshot, bounded
+ lane-compacted FP32 screening, split FP64 refine, stage II).

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

cfg = plan_config()
one = scenes(1, points=20000, frames=20, first=0, kinds=1)
with Planner(cfg, max_points=1 << 16) as p:
    x = State.from_array(one["states"][0])
    snap = p.build_snapshot(one["xyz"], x, cfg.r_max)
    r = p.plan_step(x, GoalSpec((45.0, 0.0, 2.0)), snap, None, ControlInput(9.81), 100, 1)
    print("C1 winner", r.winner, "control", r.control.vec())
S = 160
d = scenes(S, points=20000, frames=20, first=11)
with Planner(cfg, max_scenes=S, max_points=int(d["offsets"][-1])) as p:
    out = p.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"], d["seeds"])
    print("batch: planned", int((out["status"] == 0).sum()), "of", S, "winners", np.bincount(out["winner"][out["winner"] >= 0]))
