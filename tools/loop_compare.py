"""GPU closed loop vs the oracle loop: per-cycle state deviation, winner
agreement, and device loop speed."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle_py import Oracle  # noqa: E402
from test_plan_parity import make_cfg  # noqa: E402

from paper_2509_17340_b200 import ClosedLoop, Planner  # noqa: E402

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 200
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = make_cfg(4, 2, K=256, N=30, cap=7.0)
orc = Oracle()
o = orc.loop(kind, 1, orc.config(cfg), 31, capacity=10)
t0 = time.perf_counter()
o.run(cycles)
t_cpu = time.perf_counter() - t0
orecs = o.records()
planner = Planner(cfg, precision=32, max_points=10 * 7200)
loop = ClosedLoop(planner, kind, 1, 31, buffer_capacity=10, max_cycles=cycles + 10)
loop.run(2)
loop.close()
loop = ClosedLoop(planner, kind, 1, 31, buffer_capacity=10, max_cycles=cycles + 10)
t0 = time.perf_counter()
ran = loop.run(cycles)
t_gpu = time.perf_counter() - t0
grecs = loop.records()
n = min(len(orecs), len(grecs))
first_div = None
agree = 0
for i in range(n):
    dx = float(np.max(np.abs(grecs[i]["x"] - orecs[i]["x"])))
    same = grecs[i]["winner"] == orecs[i]["winner"]
    agree += same
    if first_div is None and (dx > 1e-6 or not same):
        first_div = i
    if i % 20 == 0 or i == n - 1:
        print(f"cycle {i:4d} |dx| {dx:.3e} winner {grecs[i]['winner']}/{orecs[i]['winner']} "
              f"pts {grecs[i]['n_points']}/{len(orecs[i]['cloud'])}")
print(f"cycles gpu {ran} cpu {len(orecs)}; winners agree {agree}/{n}; first divergence {first_div}")
print(f"status gpu {loop.state()[1]} cpu {o.status()}")
print(f"loop time gpu {1e3 * t_gpu / max(ran, 1):.3f} ms/cycle, cpu oracle {1e3 * t_cpu / max(len(orecs), 1):.2f} ms/cycle")
