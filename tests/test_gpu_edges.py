"""Edge cases the reference defines: empty short part, clipping at the faces,
collisions, capacity caps, forced ranks, explicit-operand API."""
import numpy as np
import pytest

import paper_1606_09218_b200 as rt
from oracle import rs_oracle as orc

pytestmark = pytest.mark.gpu


def cfg_for(n=32, b=8.0, split=7, M=15, eps=1e-8, ranks=None, max_overlap=None, kind="newton"):
    red = rt.ReductionConfig(ranks=ranks, max_sweeps=0) if ranks else \
        rt.ReductionConfig(eps=eps, max_sweeps=0)
    return rt.AssemblyConfig(grid=rt.Grid3(n, rt.Box3(b)), kernel=rt.RadialKernel(kind, 0.5), M=M,
                             split_index=split, sigma=1.0, delta=1e-6, long_format="tucker",
                             reduction=red, max_overlap=max_overlap)


def oracle_grid(pos, q, cfg, ranks):
    case = dict(kind=cfg.kernel.kind, lam=cfg.kernel.lam, b=cfg.grid.box.half_width, n=cfg.grid.n,
                M=cfg.M, split_index=cfg.split_index, delta=cfg.delta, positions=pos, charges=q)
    return orc.build_and_dense(case, ranks=ranks)["grid"]


def check(pos, q, cfg):
    res = rt.build_rs(rt.ParticleSystem(pos, q, cfg.grid.box), cfg)
    grid = rt.dense_rs(res.rs, limit=1 << 40)
    ref = oracle_grid(pos, q, cfg, tuple(res.report["tucker_ranks"]))
    assert np.max(np.abs(grid - ref)) <= 1e-10 * np.abs(ref).max()
    return res, grid


def test_particles_on_boundary_nodes(cuda):
    h = 0.5
    pos = np.array([[-7.99, -7.99, -7.99], [7.9, 7.9, 7.9], [-7.99, 7.9, 0.1], [0.0, 0.0, 7.9]])
    res, _ = check(pos, np.array([1.0, -0.5, 0.25, 0.75]), cfg_for())
    idx = res.system.indices
    assert idx.min() == 1 and idx.max() == 31


def test_single_particle(cuda):
    check(np.array([[0.3, -1.2, 2.0]]), np.array([0.7]), cfg_for(eps=1e-10))


def test_empty_short_part(cuda):
    rng = np.random.default_rng(2)
    pos = rng.uniform(-6, 6, (10, 3))
    res, _ = check(pos, rng.uniform(-1, 1, 10), cfg_for(split=15))
    assert res.rs.short.local.rank == 0 and res.gamma == 0


def test_forced_ranks(cuda):
    rng = np.random.default_rng(3)
    pos = rng.uniform(-6, 6, (30, 3))
    res, _ = check(pos, rng.uniform(-1, 1, 30), cfg_for(ranks=(5, 4, 3)))
    assert res.report["tucker_ranks"] == [5, 4, 3]


def test_collision_raises(cuda):
    pos = np.array([[0.01, 0.0, 0.0], [-0.01, 0.0, 0.0]])
    with pytest.raises(rt.ResolutionError):
        rt.build_rs(rt.ParticleSystem(pos, np.ones(2), rt.Box3(8.0)), cfg_for())


def test_overlap_cap_and_limit(cuda):
    rng = np.random.default_rng(4)
    pos = rng.uniform(-3, 3, (20, 3))
    res = rt.build_rs(rt.ParticleSystem(pos, np.ones(20), rt.Box3(8.0)), cfg_for(max_overlap=8))
    with pytest.raises(rt.CapacityError):
        rt.eval_rs_many(res.rs, res.system.indices)

def test_dense_limit_guard(cuda):
    rng = np.random.default_rng(5)
    pos = rng.uniform(-3, 3, (5, 3))
    cfg = cfg_for(n=160, b=8.0)
    res = rt.build_rs(rt.ParticleSystem(pos, np.ones(5), rt.Box3(8.0)), cfg)
    with pytest.raises(rt.CapacityError):
        rt.dense_rs(res.rs)


def test_explicit_operand_api(cuda):
    """assemble_long -> side_svd -> rhosvd (explicit side matrices on device)
    equals the shift-merged build_rs path."""
    rng = np.random.default_rng(6)
    pos = rng.uniform(-6, 6, (40, 3))
    q = rng.uniform(-1, 1, 40)
    cfg = cfg_for()
    system = rt.ParticleSystem(pos, q, cfg.grid.box)
    res = rt.build_rs(system, cfg)
    long_raw = rt.assemble_long(res.reference, res.system, cfg.split_index)
    assert long_raw.rank == 40 * (cfg.split_index + 1)
    ref_long = orc.long_side_matrices(res.reference.table, np.asarray(res.reference.tensor.weights),
                                      res.system.indices, q, cfg.split_index)
    for a, b in zip(long_raw.factors, ref_long[1]):
        assert np.array_equal(a.cpu().numpy(), b)
    t = rt.rhosvd(long_raw, cfg.reduction)
    assert list(t.ranks) == res.report["tucker_ranks"]
    d1 = t.dense(limit=1 << 30)
    d2 = res.rs.long.dense(limit=1 << 30)
    assert np.max(np.abs(d1 - d2)) <= 1e-11 * np.abs(d2).max()


def test_result_system_is_reference_type(cuda):
    """Host input -> AssemblyResult.system is the reference's host type
    (``assembly.py:271-279``): an IndexedParticleSystem with read-only numpy
    arrays that numpy code and a second build_rs accept unchanged."""
    rng = np.random.default_rng(6)
    pos = rng.uniform(-6, 6, (40, 3))
    q = rng.uniform(-1, 1, 40)
    cfg = cfg_for()
    system = rt.ParticleSystem(pos, q, cfg.grid.box)
    res = rt.build_rs(system, cfg)
    s = res.system
    assert isinstance(s, rt.IndexedParticleSystem)
    assert isinstance(s.indices, np.ndarray) and s.indices.dtype == np.int64
    assert not s.indices.flags.writeable and not s.base.positions.flags.writeable
    host = rt.snap_to_grid(system, cfg.grid)
    assert np.array_equal(s.indices, host.indices)
    assert np.array_equal(s.base.positions, host.base.positions)
    assert np.array_equal(s.charges, host.charges)
    assert s.max_displacement == host.max_displacement
    assert s.count == 40 and s.grid == cfg.grid
    # numpy code on the result, as reference users write it
    assert np.all(np.abs(s.grid.position(s.indices) - s.base.positions) == 0)
    # and it feeds back into the API (indexed input path)
    res2 = rt.build_rs(s, cfg)
    assert res2.report["tucker_ranks"] == res.report["tucker_ranks"]
    e1 = rt.reference_energy(s, res.reference)
    e2 = rt.reference_energy(host, res.reference)
    assert e1 == e2
