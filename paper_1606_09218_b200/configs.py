"""The five BASELINE.json workloads as seeded synthetic particle systems.

Recipes follow SURVEY.md section 8(d) (resolved there where BASELINE.json is
ambiguous) and are recorded in :data:`MANIFEST`:

* C1  Newton, b=10, n=128, N=64: 64 points ``U[-6,6]^3`` (seed 0, drawn as
  ``generate_random_cluster(64, Box3(6), 1e-9, seed=0, "uniform")``), charges
  ``U[-1,1]``, re-boxed to ``Box3(10)``; M=23, split 11, eps 1e-6.
* C2  Newton, b=16, n=256: 10^3 lattice, spacing 2.5, centred, jitter
  ``N(0, 0.1)`` (seed 0), charges ``(-1)^(i+j+k)``; M=27, split 13, eps 1e-6.
* C3  Newton, b=40, n=512: 10 000 points rejection-sampled in the ball of
  radius 30 with min distance 1.0 (seed 0, candidates ``U[-30,30]^3``), then
  charges: ``mix = U[0,1) < 0.7``, ``u = U[-0.5,0.5]``, ``s = choice([-1,1])``
  (three vector draws in that order); M=31, split 15, eps 1e-7.
* C4  Newton, b=64, n=1024: ``generate_random_cluster(100000, Box3(56), 0.8,
  seed=0, "uniform")`` re-boxed to ``Box3(64)``; M=35, split 17, eps 1e-7.
* C5  Yukawa lam=0.5, b=64, n=2048: 32^3 lattice, spacing 3.5, jitter
  ``N(0, 0.1)``, 1638 random vacancies (``choice(32768, 1638, replace=False)``),
  charges random sign; M=39, split 19, eps 1e-8.

All: delta = 1e-8, sigma = 1.0 (explicit; irrelevant once split_index is
fixed), max_overlap = None, long_format = "tucker", max_sweeps = 0.
"""

from __future__ import annotations

import numpy as np

from .assembly import AssemblyConfig
from .particles import Box3, Grid3, ParticleSystem, generate_random_cluster
from .quadrature import RadialKernel
from .rankred import ReductionConfig

MANIFEST = {
    "C1": dict(kernel="newton", lam=1.0, b=10.0, n=128, N=64, M=23, split_index=11, eps=1e-6),
    "C2": dict(kernel="newton", lam=1.0, b=16.0, n=256, N=1000, M=27, split_index=13, eps=1e-6),
    "C3": dict(kernel="newton", lam=1.0, b=40.0, n=512, N=10000, M=31, split_index=15, eps=1e-7),
    "C4": dict(kernel="newton", lam=1.0, b=64.0, n=1024, N=100000, M=35, split_index=17, eps=1e-7),
    "C5": dict(kernel="yukawa", lam=0.5, b=64.0, n=2048, N=31130, M=39, split_index=19, eps=1e-8),
}
DELTA = 1e-8
SIGMA = 1.0


def _c1():
    sys6 = generate_random_cluster(64, Box3(6.0), min_sep=1e-9, seed=0, charge_law="uniform")
    return sys6.positions, sys6.charges


def _lattice(d: int, spacing: float):
    ax = (np.arange(d) - (d - 1) / 2.0) * spacing
    g = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    ii, jj, kk = np.meshgrid(np.arange(d), np.arange(d), np.arange(d), indexing="ij")
    return g, (ii + jj + kk).ravel()


def _c2():
    rng = np.random.default_rng(0)
    g, parity = _lattice(10, 2.5)
    pos = g + rng.normal(0.0, 0.1, (1000, 3))
    return pos, np.where(parity % 2 == 0, 1.0, -1.0)


def _c3():
    rng = np.random.default_rng(0)
    count, radius, dmin = 10000, 30.0, 1.0
    cell = dmin
    dim = int(np.floor(2 * radius / cell))
    buckets: dict = {}
    pts = np.empty((count, 3))
    m = 0
    while m < count:
        c = rng.uniform(-radius, radius, 3)
        if not np.sqrt(np.sum(c * c)) < radius:
            continue
        key = tuple(min(dim - 1, max(0, int((c[a] + radius) / cell))) for a in range(3))
        near = []
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    near.extend(buckets.get((key[0] + dx, key[1] + dy, key[2] + dz), ()))
        if near and np.min(np.sum((pts[np.asarray(near)] - c) ** 2, axis=1)) < dmin * dmin:
            continue
        pts[m] = c
        buckets.setdefault(key, []).append(m)
        m += 1
    mix = rng.random(count) < 0.7
    u = rng.uniform(-0.5, 0.5, count)
    s = rng.choice(np.array([-1.0, 1.0]), count)
    return pts, np.where(mix, u, s)


def _c4():
    sysc = generate_random_cluster(100000, Box3(56.0), 0.8, seed=0, charge_law="uniform")
    return sysc.positions, sysc.charges


def _c5():
    rng = np.random.default_rng(0)
    g, _ = _lattice(32, 3.5)
    pos = g + rng.normal(0.0, 0.1, g.shape)
    drop = rng.choice(g.shape[0], 1638, replace=False)
    keep = np.setdiff1d(np.arange(g.shape[0]), drop)
    q = rng.integers(0, 2, size=keep.size).astype(np.float64) * 2.0 - 1.0
    return pos[keep], q


_GEN = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5}
_CACHE: dict = {}


def system(name: str) -> ParticleSystem:
    """The seeded particle system of config ``name`` (cached per process)."""
    if name not in _CACHE:
        pos, q = _GEN[name]()
        _CACHE[name] = ParticleSystem(pos, q, Box3(MANIFEST[name]["b"]))
    return _CACHE[name]


def assembly_config(name: str, ranks=None) -> AssemblyConfig:
    m = MANIFEST[name]
    red = ReductionConfig(ranks=tuple(ranks), max_sweeps=0) if ranks is not None else \
        ReductionConfig(eps=m["eps"], max_sweeps=0)
    return AssemblyConfig(grid=Grid3(m["n"], Box3(m["b"])), kernel=RadialKernel(m["kernel"], m["lam"]),
                          M=m["M"], split_index=m["split_index"], sigma=SIGMA, delta=DELTA,
                          long_format="tucker", reduction=red, max_overlap=None)


def oracle_case(name: str) -> dict:
    """Plain-array description of the config (the form ``oracle/`` consumes)."""
    m = MANIFEST[name]
    s = system(name)
    return dict(kind=m["kernel"], lam=m["lam"], b=m["b"], n=m["n"], M=m["M"],
                split_index=m["split_index"], delta=DELTA, eps=m["eps"],
                positions=np.array(s.positions), charges=np.array(s.charges))
