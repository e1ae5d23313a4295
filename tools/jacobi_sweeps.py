"""Diagnostic: rs_topeig accuracy/time vs the Jacobi sweep cap (env
RSB200_JACOBI_SWEEPS read once per process, so one cap per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.rankred import shifted_grams, top_eig, shift_histograms

# the real C2 Grams
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.assembly_config(name)
system = configs.system(name)
plan = rt.plan_for(cfg, cfg.split_index)
n = cfg.grid.n
idx = torch.tensor(rt.snap_to_grid(system, cfg.grid).indices, device="cuda")
z = torch.tensor(system.charges, device="cuda")
hist, _ = shift_histograms(idx, z, n)
G = shifted_grams(plan.table_dev, n, plan.w_long_abs, hist)
ev, U, tr = top_eig(G, 24)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    top_eig(G, 24)
e1.record()
torch.cuda.synchronize()
ref = np.load("/tmp/eig_ref.npz") if os.path.exists("/tmp/eig_ref.npz") else None
evh, Uh = ev.cpu().numpy(), U.cpu().numpy()
cap = os.environ.get("RSB200_JACOBI_SWEEPS", "16")
if ref is None:
    np.savez("/tmp/eig_ref.npz", ev=evh, U=Uh)
    print(f"sweeps {cap}: {1e3 * e0.elapsed_time(e1) / 20:.1f} us per call (reference saved)")
else:
    dev = np.max(np.abs(evh - ref["ev"]) / np.abs(ref["ev"][:, :1]))
    dU = np.max(np.abs(np.abs(np.sum(Uh[:, :12] * ref["U"][:, :12], axis=2)) - 1))
    print(f"sweeps {cap}: {1e3 * e0.elapsed_time(e1) / 20:.1f} us per call, max rel eval diff {dev:.2e}, "
          f"max |1-|cos|| of leading 12 vectors {dU:.2e}")
