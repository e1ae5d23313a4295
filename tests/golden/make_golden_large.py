"""C3-C5 golden fixtures from the REFERENCE itself.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_large.py C3
    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_large.py C5
    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_large.py C4

Writes ``tests/golden/large_<C>.npz`` and merges ``large.json``.  The GPU box
only reads those files.

* C3 (fits this 62 GB container): the reference ``build_rs`` + the FULL
  ``dense_rs`` grid (sha256, moments, per-x1-plane sums / abs sums / max,
  the x3 row sums of every (x1, x2) row, 4 full planes, 5000 samples),
  ``eval_rs_many`` at every particle node plus 2000 random points,
  ``rs_energy``, ``reference_energy``, the per-particle potential
  phi_j = P_l(x_j)/h^3 - z_j self (the ``rs_energy`` summand / z_j), and
  ``force_fd`` for EVERY particle.
* C5 (``build_rs`` peaks at ~41 GB here; the 68.7 GB grid itself does not
  fit, so no ``dense_rs``): ``eval_rs_many`` at every particle node plus
  2000 random points, the long part alone and the short part alone
  (``eval_tucker_many`` / ``eval_cct``) at 5000 random points, 4 full
  x1-planes of the Tucker part (``TuckerTensor.dense``'s contraction on the
  reference's own core and factors, one V1 row at a time; stored as a stride-8
  subsample plus row sums, column sums and the max), energies, phi and
  ``force_fd`` for EVERY particle (process pool).
* C4 (the 44 GB of side matrices plus the weighted copy do not fit): the
  reference short part (``assemble_short`` -> ``eval_cct``) at 3000 random
  points and 2000 particle nodes, and ``force_fd`` on 300 particles.  The
  long part at C4 stays pinned through the oracle (DESIGN 3).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
import warnings
from concurrent.futures import ProcessPoolExecutor

import numpy as np

import rstensor as rt  # the reference (pkg/src/rstensor)
from rstensor.formats import eval_cct, eval_rs_many, eval_tucker_many
from rstensor.observables import _long_values, force_fd, reference_energy, rs_energy

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1606_09218_b200 import configs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
PLANES = {"C3": (1, 200, 256, 511), "C4": (1, 511, 700, 1023), "C5": (1, 1023, 1500, 2047)}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_config(name):
    m = configs.MANIFEST[name]
    return rt.AssemblyConfig(grid=rt.Grid3(m["n"], rt.Box3(m["b"])),
                             kernel=rt.RadialKernel(m["kernel"], m["lam"]), M=m["M"],
                             split_index=m["split_index"], sigma=configs.SIGMA,
                             delta=configs.DELTA, long_format="tucker",
                             reduction=rt.ReductionConfig(eps=m["eps"], max_sweeps=0),
                             max_overlap=None)


def ref_system(name):
    s = configs.system(name)
    m = configs.MANIFEST[name]
    return rt.ParticleSystem(np.array(s.positions), np.array(s.charges), rt.Box3(m["b"]))


_W: dict = {}


def _force_worker_init(name):
    cfg = ref_config(name)
    indexed = rt.snap_to_grid(ref_system(name), cfg.grid)
    ref = rt.reference_for(cfg)
    import dataclasses
    _W["sys"] = indexed
    _W["ref"] = dataclasses.replace(ref, split_index=configs.MANIFEST[name]["split_index"])


def _force_chunk(js):
    return [force_fd(_W["sys"], int(j), _W["ref"]).force for j in js]


def forces(name, targets, workers=8):
    chunks = np.array_split(np.asarray(targets), max(1, 8 * workers))
    with ProcessPoolExecutor(workers, initializer=_force_worker_init, initargs=(name,)) as ex:
        out = list(ex.map(_force_chunk, chunks))
    return np.array([f for c in out for f in c]).reshape(-1, 3)


def store(name, meta, arrays):
    np.savez_compressed(os.path.join(HERE, f"large_{name}.npz"), **arrays)
    path = os.path.join(HERE, "large.json")
    allm = {}
    if os.path.exists(path):
        with open(path) as fh:
            allm = json.load(fh)
    allm[name] = meta
    with open(path, "w") as fh:
        json.dump(allm, fh, indent=1, sort_keys=True)


def phi_of(rs, res):
    h3 = res.system.grid.h ** 3
    return _long_values(rs, res.system.indices) / h3 - res.system.charges * res.reference.self_value()


def run_full(name):
    """C3: the whole reference pipeline including the dense grid."""
    t0 = time.time()
    cfg = ref_config(name)
    n = cfg.grid.n
    res = rt.build_rs(ref_system(name), cfg)
    rs = res.rs
    t_build = time.time() - t0
    grid = rt.dense_rs(rs, limit=max(n ** 3, (2 * res.gamma + 1) ** 3))
    t_dense = time.time() - t0 - t_build
    print(f"{name}: build {t_build:.1f}s dense {t_dense:.1f}s ranks={res.report['tucker_ranks']}",
          flush=True)
    rng = np.random.default_rng(11)
    rand = rng.integers(0, n, size=(2000, 3))
    pts = np.concatenate([res.system.indices, rand])
    vals = eval_rs_many(rs, pts)
    print(f"{name}: eval_rs_many {time.time() - t0:.1f}s", flush=True)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        e_rs = rs_energy(rs, res.system, res.reference)
    e_ref = reference_energy(res.system, res.reference)
    print(f"{name}: energies {time.time() - t0:.1f}s", flush=True)
    f_all = forces(name, np.arange(res.system.count))
    print(f"{name}: forces {time.time() - t0:.1f}s", flush=True)
    sample = rng.integers(0, n, size=(5000, 3))
    rep = {k: (v if not isinstance(v, np.generic) else v.item()) for k, v in res.report.items()}
    meta = dict(report=rep, ranks=list(res.report["tucker_ranks"]), gamma=res.gamma,
                rs_energy=e_rs, reference_energy=e_ref, grid_sha=sha(grid),
                grid_sum=math.fsum(grid.ravel()), grid_abs_sum=float(np.abs(grid).sum()),
                grid_sq_sum=float((grid * grid).sum()), grid_max_abs=float(np.abs(grid).max()),
                indices_sha=sha(res.system.indices), seconds=time.time() - t0)
    arrays = dict(eval_idx=pts, eval_vals=vals, phi=phi_of(rs, res), forces=f_all,
                  sample_idx=sample, sample_vals=grid[sample[:, 0], sample[:, 1], sample[:, 2]],
                  plane_sum=grid.sum(axis=(1, 2)), plane_abs_sum=np.abs(grid).sum(axis=(1, 2)),
                  plane_max_abs=np.abs(grid).max(axis=(1, 2)), row_sum=grid.sum(axis=2),
                  long_sample=eval_tucker_many(rs.long, sample))
    for p in PLANES[name]:
        arrays[f"plane_{p}"] = grid[p]
    store(name, meta, arrays)
    print(f"{name}: done {time.time() - t0:.1f}s", flush=True)


def run_reduced(name):
    """C5: the reference build_rs, point values, energies, forces, Tucker planes."""
    t0 = time.time()
    cfg = ref_config(name)
    n = cfg.grid.n
    res = rt.build_rs(ref_system(name), cfg)
    rs = res.rs
    print(f"{name}: build {time.time() - t0:.1f}s ranks={res.report['tucker_ranks']}", flush=True)
    rng = np.random.default_rng(11)
    rand = rng.integers(0, n, size=(2000, 3))
    pts = np.concatenate([res.system.indices, rand])
    vals = eval_rs_many(rs, pts)
    sample = rng.integers(0, n, size=(5000, 3))
    long_s = eval_tucker_many(rs.long, sample)
    short_s = np.array([eval_cct(rs.short, i) for i in sample])
    print(f"{name}: point values {time.time() - t0:.1f}s", flush=True)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        e_rs = rs_energy(rs, res.system, res.reference)
    phi = phi_of(rs, res)
    arrays = dict(eval_idx=pts, eval_vals=vals, phi=phi, sample_idx=sample, long_sample=long_s,
                  short_sample=short_s)
    rep = {k: (v if not isinstance(v, np.generic) else v.item()) for k, v in res.report.items()}
    meta = dict(report=rep, ranks=list(res.report["tucker_ranks"]), gamma=res.gamma,
                rs_energy=e_rs, indices_sha=sha(res.system.indices))
    store(name, meta, arrays)   # checkpoint
    # x1-planes of the Tucker part: TuckerTensor.dense's contraction
    # (formats.py:173-176) on the reference's own core and factors, one row of
    # V1 at a time (the class itself refuses a 1-row factor: rank > mode size)
    v1, v2, v3 = rs.long.factors
    # (a 2048^2 plane is 33 MB: the fixture keeps a stride-8 subsample, the
    # row and column sums -- every entry enters two of them -- and the max)
    for p in PLANES[name]:
        t = np.einsum("abc,a,jb,lc->jl", rs.long.core, v1[p], v2, v3, optimize=True)
        arrays[f"tucker_plane_{p}_sub8"] = np.ascontiguousarray(t[3::8, 5::8])
        arrays[f"tucker_plane_{p}_rowsum"] = t.sum(axis=1)
        arrays[f"tucker_plane_{p}_colsum"] = t.sum(axis=0)
        arrays[f"tucker_plane_{p}_maxabs"] = np.array(np.abs(t).max())
    store(name, meta, arrays)
    del res, rs
    idx_sys = rt.snap_to_grid(ref_system(name), cfg.grid)
    import dataclasses
    ref = dataclasses.replace(rt.reference_for(cfg), split_index=configs.MANIFEST[name]["split_index"])
    meta["reference_energy"] = reference_energy(idx_sys, ref)
    print(f"{name}: reference_energy {time.time() - t0:.1f}s", flush=True)
    arrays["forces"] = forces(name, np.arange(idx_sys.count))
    meta["seconds"] = time.time() - t0
    store(name, meta, arrays)
    print(f"{name}: done {time.time() - t0:.1f}s", flush=True)


def run_short_only(name):
    """C4: the reference short part and forces (the long part needs 59 GB)."""
    t0 = time.time()
    cfg = ref_config(name)
    n = cfg.grid.n
    m = configs.MANIFEST[name]
    idx_sys = rt.snap_to_grid(ref_system(name), cfg.grid)
    import dataclasses
    ref = dataclasses.replace(rt.reference_for(cfg), split_index=m["split_index"])
    short = rt.assemble_short(ref, idx_sys, m["split_index"], cfg.delta, cfg.overlap_policy,
                              cfg.max_overlap)
    rng = np.random.default_rng(11)
    nodes = idx_sys.indices[rng.choice(idx_sys.count, 2000, replace=False)]
    pts = np.concatenate([rng.integers(0, n, size=(3000, 3)), nodes])
    sv = np.array([eval_cct(short, i) for i in pts])
    print(f"{name}: short values {time.time() - t0:.1f}s", flush=True)
    fidx = rng.choice(idx_sys.count, 300, replace=False)
    f = forces(name, fidx)
    meta = dict(gamma=int(short.gamma), indices_sha=sha(idx_sys.indices),
                seconds=time.time() - t0)
    store(name, meta, dict(short_idx=pts, short_vals=sv, force_idx=fidx, forces=f))
    print(f"{name}: done {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        {"C3": run_full, "C5": run_reduced, "C4": run_short_only}[nm](nm)
