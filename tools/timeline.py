"""Diagnostic: kernel timeline (start/end per stream) of one prefetching C2
step from a torch profiler trace."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from torch.profiler import profile, ProfilerActivity

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
system = configs.system(name)
cfg = configs.assembly_config(name)
dp = rt.DeviceParticles(torch.tensor(system.positions, device="cuda"),
                        torch.tensor(system.charges, device="cuda"), system.box)
for _ in range(3):
    res = rt.build_rs(dp, cfg, prefetch_dense=True)
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    res = rt.build_rs(dp, cfg, prefetch_dense=True)
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True)
    torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in k)
k.sort(key=lambda e: e["ts"])
for e in k:
    print(f"{e['ts']-t0:9.1f} {e['dur']:8.1f} s{e['args'].get('stream')} {e['name'][:70]}")
cpu = [e for e in ev if e.get("cat") == "cpu_op" and e["name"] in ("aten::_local_scalar_dense", "aten::item", "aten::copy_")]
print("total span us", max(e["ts"] + e["dur"] for e in k) - t0)
