"""C5 through amppi_cycle_batch_submit / _wait at pipeline depths 1, 2, 3:
wall ms per batch (10 batches, after warm-up), alternating depths."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_17340_b200 import Planner  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

d = scenes(4096, points=20000, frames=20, first=0)
p = Planner(plan_config(), max_scenes=4096, max_points=int(d["offsets"][-1]))
pinned = torch.from_numpy(d["xyz"]).pin_memory()
args = [d["offsets"], pinned.numpy(), d["poses"], d["states"], d["goals"], d["last"]]


def sub(c):
    return p.cycle_batch_submit(*args, d["cycles"] + np.uint64(c), d["seeds"])


def run(depth, steps=10):
    t0 = time.perf_counter()
    pend = [sub(i) for i in range(min(depth - 1, steps))]
    for i in range(steps):
        if i + depth - 1 < steps:
            pend.append(sub(i + depth - 1))  # `depth` batches in flight before the wait
        p.cycle_batch_wait(pend.pop(0))
    return 1000 * (time.perf_counter() - t0) / steps


for dd in (1, 2, 3):
    run(dd, 4)
for rep in range(3):
    print(" ".join(f"depth{dd} {run(dd):.2f}" for dd in (1, 2, 3)), flush=True)
