"""Host-to-device copy bandwidth from pinned memory (the e2e floor of C5):
one 882 MB copy, the size of a C5 batch's points, best of 5."""
import torch

n = 882 * 1024 * 1024 // 4
src = torch.empty(n, dtype=torch.float32).pin_memory()
dst = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
best = 0.0
for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        dst.copy_(src, non_blocking=True)
        e1.record(s)
    s.synchronize()
    best = max(best, src.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
print(f"pinned H2D {best:.1f} GB/s ({src.numel() * 4 / 1e6:.0f} MB)")
