"""Diagnostic: which allocation calls cudaMalloc in the first step after a
synchronize (bench's step 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
system = configs.system(name)
cfg = configs.assembly_config(name)
n = cfg.grid.n
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
last = None
def step():
    global last
    last = None
    res = rt.build_rs(dp, cfg, prefetch_dense=(0, n))
    last = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(0, n))
for _ in range(8):
    step()
torch.cuda.synchronize()
torch.cuda.memory._record_memory_history(max_entries=100000)
m0 = torch.cuda.memory_stats()["num_device_alloc"]
for i in range(3):
    step()
    print("step", i, "cudaMalloc so far:", torch.cuda.memory_stats()["num_device_alloc"] - m0)
snap = torch.cuda.memory._snapshot()
for tr in snap["device_traces"]:
    for ev in tr:
        if ev["action"] in ("segment_alloc", "segment_map"):
            print(ev["action"], ev["size"], ev.get("stream"))
            for f in ev["frames"][:12]:
                print("   ", f["filename"].split("/")[-1], f["line"], f["name"])
