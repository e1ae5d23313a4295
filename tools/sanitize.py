"""compute-sanitizer target: one RS assembly (build_rs + dense_rs through the
prefetch path and the plain path), point values, energy and forces of a small
config, every short-range method.  Run as
  compute-sanitizer --tool memcheck  python tools/sanitize.py C1
  compute-sanitizer --tool racecheck python tools/sanitize.py C1"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.formats import assemble_grid

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
system, cfg = configs.system(name), configs.assembly_config(name)
res = rt.build_rs(system, cfg)
ref = None
for m in ("mma", "gemm", "l0"):
    os.environ["RSB200_SHORT"] = m
    g = assemble_grid(res.rs.long, res.rs.short)
    torch.cuda.synchronize()
    if ref is None:
        ref = g
    print(name, m, "max diff vs mma", float((g - ref).abs().max()), flush=True)
del os.environ["RSB200_SHORT"]
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
res2 = rt.build_rs(dp, cfg, prefetch_dense=True)
g2 = rt.dense_rs(res2.rs, limit=1 << 40, device=True)
torch.cuda.synchronize()
print("prefetch path diff", float((g2 - ref).abs().max()))
idx = res.system.indices
v = rt.eval_rs_many(res.rs, idx)
e = rt.rs_energy(res.rs, res.system, res.reference, check_separation=False)
f = rt.forces_fd(res.system, res.reference)
S = rt.forces_fd_scale(res.system, res.reference)
print("values", float(np.abs(v).max()), "energy", e, "forces", float(np.abs(f).max()), float(S.max()))
torch.cuda.synchronize()
print("sanitize target done")
