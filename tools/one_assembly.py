"""Diagnostic: one build_rs + dense_rs of a config (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
system = configs.system(name)
cfg = configs.assembly_config(name)
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
for _ in range(reps):
    res = rt.build_rs(dp, cfg)
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True)
    del g
torch.cuda.synchronize()
print(name, res.report["tucker_ranks"])
