"""Diagnostic: rs_topeig alone on three graded PSD matrices (C2-like n, b),
CUDA-event time per call and the per-kernel device times (torch profiler)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1606_09218_b200.rankred import top_eig

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
b = int(sys.argv[2]) if len(sys.argv) > 2 else 24
rng = np.random.default_rng(1)
gs = []
for m in range(3):
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = 10.0 ** (-np.arange(n) / (2.0 + m))
    gs.append((q * lam) @ q.T)
G = torch.tensor(np.stack(gs), device="cuda")
for _ in range(5):
    top_eig(G, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    top_eig(G, b)
e1.record()
torch.cuda.synchronize()
print(f"n={n} b={b}: rs_topeig {1e3 * e0.elapsed_time(e1) / 20:.1f} us per call (3 matrices)")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        top_eig(G, b)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
