"""Does a concurrent pinned H2D copy (the next batch's ~880 MB upload) slow the
C5 device batch?  Times cycle_batch_device alone and with the copy running on
another stream, alternating, per-kernel times included."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_17340_b200 import Planner  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

dev = torch.device("cuda", 0)
d = scenes(4096, points=20000, frames=20, first=0)
ks, cs = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
torch.cuda.set_stream(ks)
P = int(d["offsets"][-1])
p = Planner(plan_config(), max_scenes=4096, max_points=P, profile=True, stream=ks.cuda_stream)
t = {k: torch.from_numpy(np.ascontiguousarray(d[k])).to(dev) for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
t["cycles"] = torch.from_numpy(d["cycles"].view(np.int64)).to(dev)
t["seeds"] = torch.from_numpy(d["seeds"].view(np.int64)).to(dev)
ptr = {k: v.data_ptr() for k, v in t.items()}
host = torch.from_numpy(d["xyz"]).pin_memory()
dst = torch.empty_like(host, device=dev)


def run(copy: bool):
    torch.cuda.synchronize()
    p.kernel_times_reset()
    e0, e1, c0, c1 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    if copy:
        with torch.cuda.stream(cs):
            c0.record(cs)
            dst.copy_(host, non_blocking=True)
            c1.record(cs)
    e0.record(ks)
    p.cycle_batch_device(ptr, {}, 4096)
    e1.record(ks)
    torch.cuda.synchronize()
    kt = p.kernel_times()
    top = {k: round(v[0], 3) for k, v in kt.items() if v[0] > 0.3}
    return e0.elapsed_time(e1), (c0.elapsed_time(c1) if copy else 0.0), top


run(False)
for copy in (False, True, False, True, False, True):
    k, c, top = run(copy)
    print(f"copy={copy}: batch {k:.2f} ms, copy {c:.2f} ms, {top}", flush=True)
