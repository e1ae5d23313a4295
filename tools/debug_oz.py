"""Diagnostic: short-range planes [lo, hi) via DMMA vs Ozaki, tiny case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import _native as nat
from paper_1606_09218_b200.formats import assemble_grid
from oracle import rs_oracle as orc
c = orc.small_case(n=32, count=24, seed=5)
box = rt.Box3(c["b"])
cfg = rt.AssemblyConfig(grid=rt.Grid3(32, box), kernel=rt.RadialKernel("newton", 1.0), M=15,
                        split_index=7, sigma=1.0, delta=1e-6, long_format="tucker",
                        reduction=rt.ReductionConfig(eps=1e-8, max_sweeps=0), max_overlap=None)
system = rt.ParticleSystem(c["positions"], c["charges"], box)
res = rt.build_rs(system, cfg)
n = 32
for lo, hi in [(0, 32), (8, 19), (0, 11), (8, 32)]:
    outs = {}
    for s in (0, 7):
        nat.OZ_SLICES = s
        outs[s] = assemble_grid(None, res.rs.short, lo, hi).cpu().numpy()
    d = np.abs(outs[7] - outs[0])
    print(lo, hi, "max|short|", np.abs(outs[0]).max(), "max diff", d.max(),
          "worst plane", np.unravel_index(d.argmax(), d.shape))
lo, hi = 8, 32
nat.OZ_SLICES = 0
a = assemble_grid(None, res.rs.short, lo, hi).cpu().numpy()
nat.OZ_SLICES = 7
b = assemble_grid(None, res.rs.short, lo, hi).cpu().numpy()
bad = np.abs(a - b) > 1e-12
rows = np.argwhere(bad.any(axis=2))
print("bad rows (plane, x2):", len(rows), rows[:10].tolist(), "row tiles", sorted(set(((r[0] * 32 + r[1]) // 128) for r in rows)))
cols = np.argwhere(bad.any(axis=(0, 1)))
print("bad x3 cols:", cols.ravel().tolist())
for r in range(3):
    nat.OZ_SLICES = 7
    b2 = assemble_grid(None, res.rs.short, lo, hi).cpu().numpy()
    print("repeat equal:", np.array_equal(b, b2), np.abs(b2 - a).max())
