"""Diagnostic: the fused Tucker + dense-L0 pass (rs_assemble_fused_l0) vs the
two-kernel route (Tucker GEMM store, then the L0 gather accumulating) on an
x1 slab of a config: bitwise comparison and CUDA-event times.

    python tools/fused_bench.py C5 256
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs, formats
from paper_1606_09218_b200 import _native as nat

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 256
res = rt.build_rs(configs.system(name), configs.assembly_config(name))
rs = res.rs
n = rs.grid.n
lo = n // 2 - planes // 2
hi = lo + planes
out = {k: torch.empty((planes, n, n), dtype=torch.float64, device="cuda") for k in ("f", "s")}


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def run(fused, dst):
    formats._FUSED_L0 = fused
    formats.assemble_grid(rs.long, rs.short, lo, hi, out=dst)


def two_kernel(dst):
    # the build_rs prefetch route: short planes stored, Tucker part accumulated
    formats.assemble_grid(None, rs.short, lo, hi, out=dst)
    formats.tucker_accumulate(rs.long, lo, hi, dst)


tf = timed(lambda: run(True, out["f"]))
ts = timed(lambda: two_kernel(out["s"]))
modes = {}
for m in ("1", "2", "3"):
    os.environ["RSB200_FUSED_MODE"] = m
    modes[m] = timed(lambda: run(True, out["s"]))
os.environ["RSB200_FUSED_MODE"] = "0"
tl = timed(lambda: formats.assemble_grid(rs.long, None, lo, hi, out=out["s"]))
tg = timed(lambda: formats.assemble_grid(None, rs.short, lo, hi, out=out["s"]))
two_kernel(out["s"])
torch.cuda.synchronize()
same = bool(torch.equal(out["f"], out["s"]))
diff = float((out["f"] - out["s"]).abs().max() / out["s"].abs().max())
print(f"{name} planes [{lo},{hi}) ranks {rs.long.ranks}: fused {tf:.3f} ms | two-kernel "
      f"{ts:.3f} ms (tucker alone {tl:.3f}, short alone {tg:.3f}) | bitwise equal {same} "
      f"(max rel diff {diff:.2e})")
print(f"fused without gather {modes['1']:.3f} ms, without MMAs {modes['2']:.3f} ms, "
      f"neither (list build + stores) {modes['3']:.3f} ms")
print("per-plane ms: fused %.4f two-kernel %.4f" % (tf / planes, ts / planes))
