"""Probe B200 FP64 peaks and eigensolver latency (measurement helper, not product)."""
import json, os, subprocess, time
import torch

def ev_time(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3

out = {}
dev = torch.device("cuda:0")
out["gpu"] = torch.cuda.get_device_name(0)
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    t = ev_time(lambda: a @ b, iters=5)
    out[f"dgemm_{n}_tflops"] = 2 * n**3 / t / 1e12
for n in (256, 512, 1024, 2048):
    x = torch.randn(n, n, dtype=torch.float64, device=dev)
    g = x @ x.T
    t = ev_time(lambda: torch.linalg.eigh(g), iters=5, warm=2)
    out[f"eigh_{n}_ms"] = t * 1e3
    g3 = torch.stack([g, g, g])
    t = ev_time(lambda: torch.linalg.eigh(g3), iters=3, warm=1)
    out[f"eigh3_{n}_ms"] = t * 1e3
out["nproc"] = os.cpu_count()
out["lscpu"] = subprocess.run("lscpu | grep 'Model name'", shell=True, capture_output=True, text=True).stdout.strip()
out["mem"] = subprocess.run("free -g | head -2", shell=True, capture_output=True, text=True).stdout.strip()
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_fp64.json", "w"), indent=1)
