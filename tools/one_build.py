"""Diagnostic: build_rs alone (no dense grid) of a config, for a launch list:
`ncu --metrics gpu__time_duration.sum --csv python tools/one_build.py C5 2`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
system, cfg = configs.system(name), configs.assembly_config(name)
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
for _ in range(reps):
    res = rt.build_rs(dp, cfg)
torch.cuda.synchronize()
print(name, res.report["tucker_ranks"])
