"""Host-API (amppi_cycle_batch) C5 step time over pipeline chunk counts and
chunk growth ratios (schedule pipeline_chunks / pipeline_ratio), pinned
caller buffers.  Usage: python tools/pipe_sweep.py "4:1.6 8:1.1 ..." """
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_17340_b200 import Planner  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

cfg = plan_config()
data = scenes(4096, points=20000, frames=20)
planner = Planner(cfg, max_scenes=4096, max_points=int(data["offsets"][-1]))
pinned = torch.from_numpy(data["xyz"]).pin_memory()
args = [data["offsets"], pinned.numpy(), data["poses"], data["states"], data["goals"], data["last"]]
for spec in sys.argv[1].split():
    c, r = spec.split(":")
    planner.set_schedule(pipeline_chunks=int(c), pipeline_ratio=float(r))
    planner.cycle_batch(*args, data["cycles"], data["seeds"])
    best = []
    for rep in range(3):
        t0 = time.perf_counter()
        for i in range(5):
            planner.cycle_batch(*args, data["cycles"] + np.uint64(i + 1), data["seeds"])
        best.append(1000 * (time.perf_counter() - t0) / 5)
    print(f"chunks {c} ratio {r}: {min(best):.2f} ms/step (reps {' '.join(f'{b:.2f}' for b in best)})", flush=True)
