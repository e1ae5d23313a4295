"""Diagnostic: the Tucker part of one x1 slab of a config, accumulated into a
slab buffer (k_tucker_gemm_res at r3 > 32) -- for ncu:
`ncu -k regex:tucker_gemm -c 1 python tools/one_tucker.py C5 64`."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.formats import tucker_accumulate

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 64
res = rt.build_rs(configs.system(name), configs.assembly_config(name))
n = res.rs.grid.n
lo = n // 2 - planes // 2
out = torch.zeros((planes, n, n), dtype=torch.float64, device="cuda")
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tucker_accumulate(res.rs.long, lo, lo + planes, out)
    torch.cuda.synchronize()
    print(f"{name} tucker planes [{lo},{lo + planes}): {1e3 * (time.perf_counter() - t0):.3f} ms")
