"""Diagnostic: time the short-range methods (plane GEMM / L0 gather / fused
DMMA) on one x1 slab of a config and compare their results.
  python tools/short_methods.py C4 64 gemm,mma"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.formats import assemble_grid

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 64
meths = sys.argv[3].split(",") if len(sys.argv) > 3 else ["gemm", "l0", "mma"]
res = rt.build_rs(configs.system(name), configs.assembly_config(name))
n = res.rs.grid.n
planes = min(planes, n)
lo = n // 2 - planes // 2
out = torch.empty((planes, n, n), dtype=torch.float64, device="cuda")
ref = None
for m in meths:
    os.environ["RSB200_SHORT"] = m
    ts = []
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        assemble_grid(None, res.rs.short, lo, lo + planes, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    if ref is None:
        ref = out.clone()
    err = float((out - ref).abs().max() / ref.abs().max())
    print(f"{name} {m:5s} short planes [{lo},{lo + planes}) of {n}: "
          + " ".join(f"{t:.3f}" for t in ts) + f" ms -> full grid x{n / planes:.1f} = "
          f"{min(ts[1:]) * n / planes:.1f} ms (diff vs first {err:.2e})", flush=True)
