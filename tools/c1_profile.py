"""C1 latency breakdown: per-kernel device time (CUDA events) and host-to-host
p50 over 300 cycles."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

cfg = plan_config()
one = scenes(1, points=20000, frames=20, first=0, kinds=1)
x = State.from_array(one["states"][0])
goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
for prof in (False, True):
    p = Planner(cfg, precision=32, max_scenes=1, max_points=1 << 16, profile=prof)
    prev, lat = None, []
    for i in range(400):
        t0 = time.perf_counter()
        snap = p.build_snapshot(one["xyz"], x, cfg.r_max)
        r = p.plan_step(x, goal, snap, prev, la, 100 + i, 1, want_rollout=False)
        lat.append(time.perf_counter() - t0)
        prev = r.per_instance[r.winner].nominal
        if i == 99:
            p.kernel_times_reset()
            lat = []
    lat.sort()
    print(f"profile={prof}: p50 {1e3 * lat[len(lat) // 2]:.3f} ms  p99 {1e3 * lat[int(0.99 * len(lat))]:.3f} ms")
    if prof:
        kt = p.kernel_times()
        tot = 0.0
        for k, (ms, n) in sorted(kt.items(), key=lambda kv: -kv[1][0]):
            print(f"  {k:22s} {1e3 * ms / n:8.1f} us")
            tot += ms / n
        print(f"  {'sum':22s} {1e3 * tot:8.1f} us")
    p.close()
