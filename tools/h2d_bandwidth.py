"""H2D bandwidth from pinned host memory on this box: one 64.6 MB copy, and two on two streams."""
import torch, time, statistics
n = 64_600_000 // 16
h = torch.empty(n, dtype=torch.complex128).pin_memory()
d = torch.empty(n, dtype=torch.complex128, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print("H2D 64.6 MB: %.3f ms = %.1f GB/s" % (ms, 64.6e6 / ms / 1e6))
s2 = torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.complex128).pin_memory(); d2 = torch.empty_like(d)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print("2 x H2D 64.6 MB on 2 streams: %.3f ms = %.1f GB/s" % (ms, 2 * 64.6e6 / ms / 1e6))
