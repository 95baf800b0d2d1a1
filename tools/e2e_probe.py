"""Host-API (amppi_cycle_batch) step time vs pipeline chunking and host-buffer
pinning, on the C5 workload.  Usage: python tools/e2e_probe.py [scenes]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_17340_b200 import Planner  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = plan_config()
data = scenes(S, points=20000, frames=20)
planner = Planner(cfg, max_scenes=S, max_points=int(data["offsets"][-1]), profile=True)
pinned = torch.from_numpy(data["xyz"]).pin_memory()


def run(xyz, steps=5):
    args = [data[k] for k in ("offsets",)] + [xyz] + [data[k] for k in ("poses", "states", "goals", "last")]
    planner.cycle_batch(*args, data["cycles"], data["seeds"])
    t0 = time.perf_counter()
    for i in range(steps):
        planner.cycle_batch(*args, data["cycles"] + np.uint64(i + 1), data["seeds"])
    return 1000 * (time.perf_counter() - t0) / steps


for chunks in ("1", "2", "4", "8"):
    planner.set_schedule(pipeline_chunks=int(chunks))
    planner.kernel_times_reset()
    t = run(pinned.numpy())
    kt = planner.kernel_times()
    ks = " ".join(f"{k}={v[0] / 6:.2f}" for k, v in sorted(kt.items()))
    print(f"chunks {chunks}: pinned {t:.2f} ms | {ks}", flush=True)
