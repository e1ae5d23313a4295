"""Diagnostic: host-time between trace points of _build_rs (RSB200_HOST_TRACE=1)."""
import os, sys, time
os.environ["RSB200_HOST_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs, assembly

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
system = configs.system(name)
cfg = configs.assembly_config(name)
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
n = cfg.grid.n
acc = {}
for it in range(25):
    torch.cuda.synchronize()
    assembly._TRACE.clear()
    assembly._mark("call")
    res = rt.build_rs(dp, cfg, prefetch_dense=(0, n))
    assembly._mark("built")
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(0, n))
    assembly._mark("dense")
    torch.cuda.synchronize()
    assembly._mark("synced")
    if it >= 5:
        tr = assembly._TRACE
        for (a, ta), (b, tb) in zip(tr[:-1], tr[1:]):
            acc.setdefault(f"{a}->{b}", []).append(1e6 * (tb - ta))
for k, v in acc.items():
    print(f"{k:22s} {np.median(v):8.1f} us")
print("total", sum(np.median(v) for v in acc.values()))
print("front pool:", {k: len(v["bufs"]) for k, v in assembly._FRONT_POOL.items()})
