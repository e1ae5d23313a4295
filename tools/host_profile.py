"""Diagnostic: host (Python) time per RS step, by function (cProfile), for the
prefetching bench step -- shows how long the host takes to enqueue work."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
system = configs.system(name)
cfg = configs.assembly_config(name)
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
n = cfg.grid.n
for _ in range(5):
    res = rt.build_rs(dp, cfg, prefetch_dense=(0, n))
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(0, n))
torch.cuda.synchronize()
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    res = rt.build_rs(dp, cfg, prefetch_dense=(0, n))
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(0, n))
    torch.cuda.synchronize()
print(f"wall per step {1e3 * (time.perf_counter() - t0) / reps:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    res = rt.build_rs(dp, cfg, prefetch_dense=(0, n))
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(0, n))
    torch.cuda.synchronize()
pr.disable()
st = io.StringIO()
pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(40)
print(st.getvalue()[:9000])
