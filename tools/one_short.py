"""Diagnostic: the short-range assembly of one x1 slab of a config (for ncu:
`ncu -k regex:short -s 1 -c 1 python tools/one_short.py C5 64`)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.formats import assemble_grid

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 64
res = rt.build_rs(configs.system(name), configs.assembly_config(name))
n = res.rs.grid.n
lo = n // 2 - planes // 2
out = torch.empty((planes, n, n), dtype=torch.float64, device="cuda")
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else [None]
ref = None
for v in variants:
    if v is not None:
        os.environ["RSB200_L0_VARIANT"] = v
    ts = []
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assemble_grid(None, res.rs.short, lo, lo + planes, out=out)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    if ref is None:
        ref = out.clone()
    err = float((out - ref).abs().max() / ref.abs().max())
    print(f"{name} variant {v} short planes [{lo},{lo + planes}): "
          + " ".join(f"{t:.3f}" for t in ts) + f" ms  (diff vs first {err:.2e})")
