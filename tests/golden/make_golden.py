"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Outputs ``tests/golden/*.npz`` + ``golden.json``.  The GPU box never runs this
script (the reference is not there); tests only read the committed outputs.
Inputs come from ``paper_1606_09218_b200.configs`` (seeded recipes) so the
same systems are used by the tests and the bench.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
import warnings

import numpy as np

import rstensor as rt  # the reference (pkg/src/rstensor)
from rstensor.formats import eval_rs_many
from rstensor.observables import force_fd, reference_energy, rs_energy

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1606_09218_b200 import configs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT: dict = {}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_config(kind, lam, b, n, M, split, delta, eps=None, ranks=None):
    red = rt.ReductionConfig(ranks=ranks, max_sweeps=0) if ranks else \
        rt.ReductionConfig(eps=eps, max_sweeps=0)
    return rt.AssemblyConfig(grid=rt.Grid3(n, rt.Box3(b)), kernel=rt.RadialKernel(kind, lam), M=M,
                             split_index=split, sigma=1.0, delta=delta, long_format="tucker",
                             reduction=red, max_overlap=None)


def prologue(name, kind, lam, b, n, M, split, delta):
    cfg = ref_config(kind, lam, b, n, M, split, delta, eps=1e-6)
    ref = rt.reference_for(cfg)
    short, _ = rt.split_tensor(ref, split)
    gamma = rt.effective_support(short, delta, ref.grid.h)
    import dataclasses
    ref_s = dataclasses.replace(ref, split_index=split)
    OUT[f"prologue_{name}"] = dict(
        table_sha=sha(ref.tensor.factors[0]), weights_sha=sha(ref.tensor.weights),
        nodes_sha=sha(ref.rule.nodes), qweights_sha=sha(ref.rule.weights), gamma=int(gamma),
        self_value=ref_s.self_value(), h_M=ref.rule.h_M, R=ref.R)
    np.savez(os.path.join(HERE, f"prologue_{name}.npz"), nodes=ref.rule.nodes,
             qweights=ref.rule.weights, weights=ref.tensor.weights,
             table_rows=ref.tensor.factors[0][:: max(1, (2 * n) // 64)])


def full_case(name, kind, lam, b, n, M, split, delta, eps, positions, charges, n_eval=400,
              n_force=8, full_grid=False, planes=(), seed=1):
    t0 = time.time()
    system = rt.ParticleSystem(positions, charges, rt.Box3(b))
    cfg = ref_config(kind, lam, b, n, M, split, delta, eps=eps)
    res = rt.build_rs(system, cfg)
    rs = res.rs
    grid = rt.dense_rs(rs, limit=max(n ** 3, (2 * res.gamma + 1) ** 3))
    rng = np.random.default_rng(seed)
    pts = rng.integers(0, n, size=(n_eval, 3))
    pts = np.concatenate([pts, res.system.indices[: min(50, res.system.count)]])
    vals = eval_rs_many(rs, pts)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        e_rs = rs_energy(rs, res.system, res.reference)
    e_ref = reference_energy(res.system, res.reference)
    fidx = np.linspace(0, res.system.count - 1, min(n_force, res.system.count)).astype(int)
    forces = np.array([force_fd(res.system, int(j), res.reference).force for j in fidx])
    spec = rt.side_svd(rt.assemble_long(res.reference, res.system, split))
    sample = rng.integers(0, n, size=(5000, 3))
    rep = {k: (v if not isinstance(v, np.generic) else v.item()) for k, v in res.report.items()}
    OUT[f"case_{name}"] = dict(
        report=rep, ranks=list(res.report["tucker_ranks"]), gamma=res.gamma,
        rs_energy=e_rs, reference_energy=e_ref, grid_sum=float(grid.sum()),
        grid_abs_sum=float(np.abs(grid).sum()), grid_sq_sum=float((grid * grid).sum()),
        grid_max_abs=float(np.abs(grid).max()), grid_sha=sha(grid), indices_sha=sha(res.system.indices),
        seconds=time.time() - t0)
    arrays = dict(eval_idx=pts, eval_vals=vals, force_idx=fidx, forces=forces,
                  sample_idx=sample, sample_vals=grid[sample[:, 0], sample[:, 1], sample[:, 2]],
                  indices=res.system.indices, spectrum0=spec.values[0][:64],
                  spectrum1=spec.values[1][:64], spectrum2=spec.values[2][:64],
                  long_sample=rs.long.dense(limit=n ** 3)[sample[:, 0], sample[:, 1], sample[:, 2]])
    for p in planes:
        arrays[f"plane_{p}"] = grid[p]
    if full_grid:
        arrays["grid"] = grid
    np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), **arrays)
    print(f"{name}: {time.time() - t0:.1f}s ranks={res.report['tucker_ranks']} gamma={res.gamma}",
          flush=True)


def tiny(kind):
    rng = np.random.default_rng(5)
    n, b, count = 32, 8.0, 24
    h = 2 * b / n
    while True:
        pos = rng.uniform(-0.7 * b, 0.7 * b, (count, 3))
        idx = np.clip(np.ceil(pos / h + n // 2 - 0.5).astype(np.int64), 1, n - 1)
        if np.unique(idx, axis=0).shape[0] == count:
            break
    q = rng.uniform(-1.0, 1.0, count)
    return pos, q


def main():
    for name, m in configs.MANIFEST.items():
        prologue(name, m["kernel"], m["lam"], m["b"], m["n"], m["M"], m["split_index"],
                 configs.DELTA)
    prologue("tiny_newton", "newton", 1.0, 8.0, 32, 15, 7, 1e-6)
    prologue("tiny_yukawa", "yukawa", 0.5, 8.0, 32, 15, 7, 1e-6)
    prologue("slater48", "slater", 1.5, 10.0, 48, 17, 8, 1e-6)

    # generators: the package's seeded recipes vs the reference generators
    c1 = rt.generate_random_cluster(64, rt.Box3(6.0), min_sep=1e-9, seed=0, charge_law="uniform")
    c4s = rt.generate_random_cluster(3000, rt.Box3(56.0), 0.8, seed=0, charge_law="uniform")
    lat = rt.generate_lattice((7, 5, 3), 1.25, charge_law="random_sign", seed=3)
    OUT["generators"] = dict(c1_pos=sha(c1.positions), c1_q=sha(c1.charges),
                             c4_3000_pos=sha(c4s.positions), c4_3000_q=sha(c4s.charges),
                             lattice_pos=sha(lat.positions), lattice_q=sha(lat.charges))
    for name in ("C2", "C3", "C5"):
        s = configs.system(name)
        m = configs.MANIFEST[name]
        snapped = rt.snap_to_grid(rt.ParticleSystem(s.positions, s.charges, rt.Box3(m["b"])),
                                  rt.Grid3(m["n"], rt.Box3(m["b"])))
        OUT[f"snap_{name}"] = dict(indices=sha(snapped.indices), positions=sha(snapped.base.positions),
                                   max_disp=snapped.max_displacement, count=snapped.count,
                                   pos_sha=sha(s.positions), q_sha=sha(s.charges))

    for kind in ("newton", "yukawa"):
        pos, q = tiny(kind)
        full_case(f"tiny_{kind}", kind, 0.5 if kind == "yukawa" else 1.0, 8.0, 32, 15, 7, 1e-6,
                  1e-8, pos, q, n_force=24, full_grid=True)
    for name, extra in (("C1", dict(planes=(1, 64))), ("C2", dict(planes=(128,)))):
        m = configs.MANIFEST[name]
        s = configs.system(name)
        full_case(name, m["kernel"], m["lam"], m["b"], m["n"], m["M"], m["split_index"],
                  configs.DELTA, m["eps"], s.positions, s.charges, **extra)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(OUT, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
