"""Host-API (amppi_cycle_batch) C5 step with the pipeline trace on: prints the
upload / compute event timeline (ms from the first copy) of each chunk."""
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
pinned = torch.from_numpy(data["xyz"]).pin_memory()
args = [data["offsets"], pinned.numpy(), data["poses"], data["states"], data["goals"], data["last"]]
for spec in (sys.argv[1:] or ["6:1.2"]):
    c, r = spec.split(":")
    p = Planner(cfg, max_scenes=4096, max_points=int(data["offsets"][-1]), pipeline_chunks=int(c),
                pipeline_ratio=float(r))
    for i in range(3):
        p.cycle_batch(*args, data["cycles"] + np.uint64(i), data["seeds"])
    p.set_schedule(trace=1)
    t0 = time.perf_counter()
    p.cycle_batch(*args, data["cycles"] + np.uint64(9), data["seeds"])
    print(f"chunks {c} ratio {r}: host {1000 * (time.perf_counter() - t0):.2f} ms", flush=True)
    p.set_schedule(trace=0)
    ts = []
    for i in range(5):
        t0 = time.perf_counter()
        p.cycle_batch(*args, data["cycles"] + np.uint64(20 + i), data["seeds"])
        ts.append(1000 * (time.perf_counter() - t0))
    print(f"   untraced: {' '.join(f'{t:.2f}' for t in ts)}", flush=True)
    p.close()
