"""Diagnostic: can the fused DMMA short kernel (SM-issue / shared-memory bound) and
the dense-L0 gather (L2-read bound) share the SMs?  Planes [lo, lo+a) by the fused
kernel on one stream, [lo+a, lo+P) by the gather on another, timed together.
  python tools/corun.py C5 64 32"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.formats import assemble_grid

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 64
splits = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "32").split(",")]
res = rt.build_rs(configs.system(name), configs.assembly_config(name))
n = res.rs.grid.n
lo = n // 2 - P // 2
out = torch.empty((P, n, n), dtype=torch.float64, device="cuda")
ref = torch.empty_like(out)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(method, a, b, dst, slot):
    os.environ["RSB200_SHORT"] = method
    assemble_grid(None, res.rs.short, lo + a, lo + b, out=dst[a:b], workspace_slot=slot)


def timed(fn, reps=4):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:])


t_m = timed(lambda: run("mma", 0, P, ref, "assemble"))
print(f"{name} {P} planes: mma alone {t_m:.3f} ms", flush=True)
t_l = timed(lambda: run("l0", 0, P, out, "assemble"))
print(f"  l0 alone {t_l:.3f} ms (diff {float((out - ref).abs().max() / ref.abs().max()):.1e})", flush=True)
for pad in os.environ.get("CORUN_PADS", "0,64").split(","):
    os.environ["RSB200_MMA_PAD_KB"] = pad
    t_mp = timed(lambda: run("mma", 0, P, out, "assemble"))
    for a in splits:
        def both():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                run("mma", 0, a, out, "assemble")
            with torch.cuda.stream(s2):
                run("l0", a, P, out, "assemble_side")
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        out.zero_()
        t = timed(both)
        err = float((out - ref).abs().max() / ref.abs().max())
        print(f"  pad {pad} KB (mma alone {t_mp:.3f}): mma [0,{a}) || l0 [{a},{P}): {t:.3f} ms (diff {err:.1e})", flush=True)
