"""Diagnostic: device->host bandwidth into pinned memory (one copy / chunked / 2 streams)."""
import torch, time
n = 134217728 // 8
d = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for _ in range(3):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
print(f"single copy {t:.3f} ms  {134.217728 / t:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
half = n // 2
with torch.cuda.stream(s1):
    h[:half].copy_(d[:half], non_blocking=True)
with torch.cuda.stream(s2):
    h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize()
t = (time.perf_counter() - t0) * 1e3
print(f"two streams {t:.3f} ms  {134.217728 / t:.1f} GB/s")
hp = torch.empty(n, dtype=torch.float64)
t0 = time.perf_counter(); hp.copy_(d); torch.cuda.synchronize()
t = (time.perf_counter() - t0) * 1e3
print(f"pageable {t:.3f} ms  {134.217728 / t:.1f} GB/s")
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
e0.record(); d.copy_(h2, non_blocking=True); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
print(f"H2D single {t:.3f} ms  {134.217728 / t:.1f} GB/s")
