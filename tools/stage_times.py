"""Diagnostic: wall-clock breakdown of one RS assembly step (synchronising
between stages -- NOT a bench number)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs, _native as nat
from paper_1606_09218_b200.formats import assemble_grid

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
system = configs.system(name)
cfg = configs.assembly_config(name)
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
n = cfg.grid.n
out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    res = rt.build_rs(dp, cfg)
    assemble_grid(res.rs.long, res.rs.short, out=out)
torch.cuda.synchronize()
L = nat.lib()
reps = 10
t0 = time.perf_counter()
for _ in range(reps):
    res = rt.build_rs(dp, cfg)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(reps):
    assemble_grid(res.rs.long, res.rs.short, out=out)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{name}: build_rs {1e3*(t1-t0)/reps:.3f} ms   assemble {1e3*(t2-t1)/reps:.3f} ms")
L.rs_prof_enable(1)
for _ in range(reps):
    res = rt.build_rs(dp, cfg)
    assemble_grid(res.rs.long, res.rs.short, out=out)
torch.cuda.synchronize()
L.rs_prof_enable(0)
for k in ("topeig", "syrk", "shift_project", "core", "short_rows", "gemm_plane", "gemm_short", "gemm_tucker", "oz_mma", "short_l0", "tucker_f"):
    ms, c = nat.prof_query(k)
    print(f"  {k:14s} {ms/reps:.4f} ms/step  ({c/reps:.0f} launches)")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        res = rt.build_rs(dp, cfg)
        assemble_grid(res.rs.long, res.rs.short, out=out)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))

import cProfile, pstats, io
pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
for _ in range(10):
    res = rt.build_rs(dp, cfg, prefetch_dense=True)
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True)
torch.cuda.synchronize()
pr.disable()
st = io.StringIO()
pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(25)
print(st.getvalue()[:6000])
