"""Diagnostic: the prefetch route's two kernels on an x1 slab -- short planes
(dense-L0 gather) then the Tucker part accumulated -- sequential vs pipelined
in G plane groups on two streams (the Tucker part of group g behind the short
part of group g, concurrent with the short part of group g+1).

    python tools/overlap_bench.py C5 256 8
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs, formats

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 256
groups = [int(g) for g in (sys.argv[3] if len(sys.argv) > 3 else "2,4,8,16").split(",")]
res = rt.build_rs(configs.system(name), configs.assembly_config(name))
rs = res.rs
n = rs.grid.n
lo = n // 2 - planes // 2
hi = lo + planes
out = torch.empty((planes, n, n), dtype=torch.float64, device="cuda")
ref = torch.empty_like(out)
s_short = torch.cuda.Stream()
s_tuck = torch.cuda.Stream()


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def sequential(dst):
    formats.assemble_grid(None, rs.short, lo, hi, out=dst)
    formats.tucker_accumulate(rs.long, lo, hi, dst)


def pipelined(dst, G):
    cur = torch.cuda.current_stream()
    s_short.wait_stream(cur)
    s_tuck.wait_stream(cur)
    step = -(-planes // G)
    evs = []
    with torch.cuda.stream(s_short):
        for g0 in range(0, planes, step):
            g1 = min(planes, g0 + step)
            formats.assemble_grid(None, rs.short, lo + g0, lo + g1, out=dst[g0:g1],
                                  workspace_slot="assemble_side")
            e = torch.cuda.Event()
            e.record(s_short)
            evs.append((g0, g1, e))
    with torch.cuda.stream(s_tuck):
        for g0, g1, e in evs:
            s_tuck.wait_event(e)
            formats.tucker_accumulate(rs.long, lo + g0, lo + g1, dst[g0:g1])
    cur.wait_stream(s_short)
    cur.wait_stream(s_tuck)


ts = timed(lambda: sequential(ref))
print(f"{name} planes [{lo},{hi}): sequential {ts:.3f} ms")
for G in groups:
    tp = timed(lambda: pipelined(out, G))
    same = bool(torch.equal(out, ref))
    print(f"  pipelined G={G}: {tp:.3f} ms  bitwise equal {same}")
