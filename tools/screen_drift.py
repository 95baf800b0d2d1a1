"""Whole-batch FP32-screening drift (amppi_screen_drift) on the C5 batch and
on C4-sized instances; prints one JSON line per case.

  python tools/screen_drift.py [scenes=4096] [stride=1]

Each case: cycle_batch_device over the scenes, then every stride-th sample of
every instance integrated as the screening does (FP32) and as the refine does
(FP64), compared step by step (tests/test_screen_drift.py asserts the same)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_17340_b200 import Planner  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402


def run(name, cfg, n, first, stride):
    d = scenes(n, points=20000, frames=20, first=first)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(d[k])).to(dev)
         for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
    t["cycles"] = torch.from_numpy(d["cycles"].view(np.int64)).to(dev)
    t["seeds"] = torch.from_numpy(d["seeds"].view(np.int64)).to(dev)
    ptr = {k: v.data_ptr() for k, v in t.items()}
    with Planner(cfg, max_scenes=n, max_points=int(d["offsets"][-1])) as p:
        p.cycle_batch_device(ptr, {}, n)
        p.synchronize()
        r = p.screen_drift(ptr, n, 0, stride)
    band = 1e-4 * cfg.weights.collision.d_max + 1e-4
    r.update(case=name, scenes=n, sample_stride=stride, band_m=band,
             clearance_diff_over_band=r["max_clearance_diff"] / band)
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    stride = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    run("C5 4096-scene batch (forest / verticals / inclines), 4x2 x 256 x 30", plan_config(), n, 0, stride)
    run("C4-sized instances, 8x8 x 8192 x 50 (every 4th sample)", plan_config(8, 8, K=8192, N=50), 8, 4096, 4)
    run("the paper's default ensemble, 5x3 x 256 x 25, 1024 scenes", plan_config(5, 3, K=256, N=25), 1024, 8192, 1)
