"""Per-kernel device time of the C1 plan cycle (one 20k-point forest scene,
4x2 anchors x 256 samples x 30 steps) through the C-ABI with CUDA-event
profiling on, plus host-to-host wall time per call."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402


def main(cycles=300):
    cfg = plan_config()
    one = scenes(1, points=20000, frames=20, first=0, kinds=1)
    x = State.from_array(one["states"][0])
    goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
    la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
    out = {}
    for prof in (False, True):
        p = Planner(cfg, precision=32, max_scenes=1, max_points=1 << 16, profile=prof)
        prev, snap_ms, plan_ms = None, [], []
        for i in range(cycles + 50):
            t0 = time.perf_counter()
            snap = p.build_snapshot(one["xyz"], x, cfg.r_max)
            t1 = time.perf_counter()
            r = p.plan_step(x, goal, snap, prev, la, 100 + i, 1, want_rollout=False)
            t2 = time.perf_counter()
            prev = r.per_instance[r.winner].nominal
            if i == 49 and prof:
                p.kernel_times_reset()
            if i >= 50:
                snap_ms.append(1e3 * (t1 - t0))
                plan_ms.append(1e3 * (t2 - t1))
        snap_ms.sort()
        plan_ms.sort()
        key = "profiled" if prof else "plain"
        out[key] = {"snapshot_p50_ms": snap_ms[len(snap_ms) // 2], "plan_p50_ms": plan_ms[len(plan_ms) // 2]}
        if prof:
            out["kernels_us_per_cycle"] = {k: round(1e3 * v[0] / cycles, 2) for k, v in p.kernel_times().items()}
        p.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
