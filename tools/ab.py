"""A/B timing of library variants on the C5 device step (per-kernel CUDA-event
times, the batch as one chunk), alternating variants to cancel drift.

  python tools/ab.py base:build_var/base/libamppi_b200.so new:paper_2509_17340_b200/libamppi_b200.so [reps]

Each measurement runs in its own process (one library per process)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.environ["AB_ROOT"])
import numpy as np, torch
from paper_2509_17340_b200 import Planner
from paper_2509_17340_b200.workloads import plan_config, scenes
cfg = plan_config()
d = scenes(4096, points=20000, frames=20, first=0)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
P = int(d["offsets"][-1])
p = Planner(cfg, max_scenes=4096, max_points=P, profile=True, stream=st.cuda_stream, device_chunks=1)
t = {k: torch.from_numpy(np.ascontiguousarray(d[k])).to(dev) for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
t["cycles"] = torch.from_numpy(d["cycles"].view(np.int64)).to(dev)
t["seeds"] = torch.from_numpy(d["seeds"].view(np.int64)).to(dev)
ptr = {k: v.data_ptr() for k, v in t.items()}
out = {"status": torch.zeros(4096, dtype=torch.int32, device=dev)}
optr = {k: v.data_ptr() for k, v in out.items()}
for i in range(3):
    t["cycles"].add_(1); p.cycle_batch_device(ptr, optr, 4096, cfg.r_max)
p.synchronize(); p.kernel_times_reset()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(5):
    t["cycles"].add_(1); p.cycle_batch_device(ptr, optr, 4096, cfg.r_max)
e1.record(st); p.synchronize()
kt = p.kernel_times()
print(json.dumps({"step_ms": e0.elapsed_time(e1) / 5, "ok": int((out["status"] == 0).sum()),
                  "kernels": {k: v[0] / v[1] for k, v in kt.items()}}))
'''


def main():
    variants = [a.split(":", 1) for a in sys.argv[1:] if ":" in a]
    reps = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 3
    res = {name: [] for name, _ in variants}
    for r in range(reps):
        for name, lib in variants:
            env = dict(os.environ, AB_ROOT=ROOT, AMPPI_LIB_PATH=os.path.join(ROOT, lib), AMPPI_ABI_LENIENT="1")
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print(name, "FAILED", out.stderr[-2000:], flush=True)
                continue
            d = json.loads(line[-1])
            res[name].append(d)
            print(name, r, round(d["step_ms"], 3), d["ok"], {k: round(v, 3) for k, v in sorted(d["kernels"].items())},
                  flush=True)
    print("\nmedians:")
    for name, runs in res.items():
        if not runs:
            continue
        keys = sorted(runs[0]["kernels"])
        med = lambda xs: sorted(xs)[len(xs) // 2]
        print(name, "step", round(med([x["step_ms"] for x in runs]), 3),
              {k: round(med([x["kernels"].get(k, 0) for x in runs]), 3) for k in keys})


if __name__ == "__main__":
    main()
