"""Does a host->device copy on one stream slow kernels on another?  Times a
compute loop (torch bf16 matmuls, then the planner's device batch) alone and
with a concurrent pinned H2D copy of ~880 MB."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

dev = torch.device("cuda", 0)
cs, ks = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
host = torch.empty(220_000_000, dtype=torch.float32).pin_memory()
dst = torch.empty_like(host, device=dev)
a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)


def compute(n=40):
    with torch.cuda.stream(ks):
        for _ in range(n):
            a @ a


def timed(copy: bool):
    torch.cuda.synchronize()
    e0, e1, c0, c1 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    t0 = time.perf_counter()
    if copy:
        with torch.cuda.stream(cs):
            c0.record(cs)
            dst.copy_(host, non_blocking=True)
            c1.record(cs)
    e0.record(ks)
    compute()
    e1.record(ks)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (c0.elapsed_time(c1) if copy else 0.0), 1000 * (time.perf_counter() - t0)


timed(False)
for copy in (False, True, False, True):
    k, c, w = timed(copy)
    print(f"copy={copy}: compute {k:.2f} ms, copy {c:.2f} ms, wall {w:.2f} ms", flush=True)
