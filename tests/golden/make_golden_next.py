"""Golden fixtures for the SURVEY §8(f) "next" rows, from the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_next.py

(1) ALS refinement (``c2t_als`` with ``max_sweeps=3``, the reference default),
(2) the canonical long format (``tucker_to_canonical``; ``build_rs``'s default
``long_format``), (3) the ``rs-tensor-container v1`` files written by the
reference's ``write_rs`` / ``write_reference``.  Outputs ``next_*.npz``,
``next_*.rsc`` and ``next.json``; the GPU box only reads them.
"""

from __future__ import annotations

import json
import os
import sys
import warnings

import numpy as np

import rstensor as rt  # the reference (pkg/src/rstensor)
from rstensor.container import write_reference, write_rs
from rstensor.formats import eval_rs_many
from rstensor.observables import grad_long, rs_energy

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from make_golden import sha, tiny  # noqa: E402
from paper_1606_09218_b200 import configs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cfg_for(n, b, M, split, kind, lam, delta, eps, sweeps, fmt):
    # reduce_long=True: the canonical format goes through RHOSVD/ALS and
    # tucker_to_canonical even below the reduce threshold
    return rt.AssemblyConfig(grid=rt.Grid3(n, rt.Box3(b)), kernel=rt.RadialKernel(kind, lam), M=M,
                             split_index=split, sigma=1.0, delta=delta, long_format=fmt,
                             reduction=rt.ReductionConfig(eps=eps, max_sweeps=sweeps),
                             max_overlap=None, reduce_long=True)


def case(name, system, cfg, n_eval=300, seed=2):
    res = rt.build_rs(system, cfg)
    n = cfg.grid.n
    grid = rt.dense_rs(res.rs, limit=max(n ** 3, (2 * res.gamma + 1) ** 3))
    rng = np.random.default_rng(seed)
    pts = np.concatenate([rng.integers(0, n, size=(n_eval, 3)), res.system.indices[:40]])
    vals = eval_rs_many(res.rs, pts)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        e = rs_energy(res.rs, res.system, res.reference)
    rep = {k: (v if not isinstance(v, np.generic) else v.item()) for k, v in res.report.items()}
    meta = dict(report=rep, rs_energy=e, grid_max_abs=float(np.abs(grid).max()), grid_sha=sha(grid))
    arrays = dict(eval_idx=pts, eval_vals=vals)
    if n <= 64:
        arrays["grid"] = grid
    else:
        sample = rng.integers(0, n, size=(6000, 3))
        arrays.update(sample_idx=sample, sample_vals=grid[sample[:, 0], sample[:, 1], sample[:, 2]])
    np.savez_compressed(os.path.join(HERE, f"next_{name}.npz"), **arrays)
    print(name, rep.get("tucker_ranks"), rep.get("reduced_canonical_rank"), flush=True)
    return res, meta


def main():
    out = {}
    pos, q = tiny("newton")
    tiny_sys = rt.ParticleSystem(pos, q, rt.Box3(8.0))
    cfg = cfg_for(32, 8.0, 15, 7, "newton", 1.0, 1e-6, 1e-8, 3, "tucker")
    res, out["tiny_tucker_als3"] = case("tiny_tucker_als3", tiny_sys, cfg)
    write_rs(res.rs, os.path.join(HERE, "next_tiny_tucker.rsc"))
    # grad_long of the reference's own RS tensor: the
    # container above carries its inputs, these are its dense components
    comps = grad_long(res.rs)
    np.savez_compressed(os.path.join(HERE, "next_tiny_grad.npz"),
                        **{f"g{a}": c.dense(limit=32 ** 3) for a, c in enumerate(comps)})
    ref = rt.reference_for(cfg_for(32, 8.0, 15, 7, "newton", 1.0, 1e-6, 1e-8, 0, "tucker"))
    write_reference(ref, os.path.join(HERE, "next_tiny_reference.rsc"))
    m = configs.MANIFEST["C1"]
    s0 = configs.system("C1")
    s = rt.ParticleSystem(s0.positions, s0.charges, rt.Box3(m["b"]))
    # the canonical RS container requires 2 gamma + 1 <= n: C1 at delta = 1e-4 (gamma 48)
    for fmt, delta, sweeps in (("tucker", configs.DELTA, 3), ("canonical", 1e-4, 0),
                               ("canonical", 1e-4, 3)):
        cfg = cfg_for(m["n"], m["b"], m["M"], m["split_index"], m["kernel"], m["lam"], delta,
                      m["eps"], sweeps, fmt)
        name = f"C1_{fmt}_als{sweeps}"
        res, out[name] = case(name, s, cfg)
        if fmt == "canonical" and sweeps == 3:
            write_rs(res.rs, os.path.join(HERE, "next_C1_canonical.rsc"))
            comps = grad_long(res.rs)
            rng = np.random.default_rng(7)
            smp = rng.integers(0, m["n"], size=(4000, 3))
            np.savez_compressed(os.path.join(HERE, "next_C1_canonical_grad.npz"), sample_idx=smp,
                                **{f"g{a}": c.dense(limit=m["n"] ** 3)[smp[:, 0], smp[:, 1], smp[:, 2]]
                                   for a, c in enumerate(comps)})
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".rsc"):
            with open(os.path.join(HERE, f), "rb") as fh:
                out[f"file_{f}"] = dict(sha=sha(np.frombuffer(fh.read(), np.uint8)))
    with open(os.path.join(HERE, "next.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
