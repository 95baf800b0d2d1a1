"""A few C1 plan cycles (for ncu captures of the latency-mode kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

cfg = plan_config()
one = scenes(1, points=20000, frames=20, first=0, kinds=1)
x = State.from_array(one["states"][0])
goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
p = Planner(cfg, precision=32, max_scenes=1, max_points=1 << 16)
prev = None
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    snap = p.build_snapshot(one["xyz"], x, cfg.r_max)
    r = p.plan_step(x, goal, snap, prev, la, 100 + i, 1, want_rollout=False)
    prev = r.per_instance[r.winner].nominal
print("ok", r.winner)
