"""Host prologue of the package vs the reference's own outputs (golden), bit-exact.

Golden hashes were produced by running the reference (tests/golden/make_golden.py);
equality of sha256 over the raw float64 bytes means bit-identical arrays.
"""
import dataclasses
import hashlib

import numpy as np
import pytest

import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from conftest import load_npz


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


PROLOGUES = {
    **{k: (m["kernel"], m["lam"], m["b"], m["n"], m["M"], m["split_index"], configs.DELTA)
       for k, m in configs.MANIFEST.items()},
    "tiny_newton": ("newton", 1.0, 8.0, 32, 15, 7, 1e-6),
    "tiny_yukawa": ("yukawa", 0.5, 8.0, 32, 15, 7, 1e-6),
    "slater48": ("slater", 1.5, 10.0, 48, 17, 8, 1e-6),
}


@pytest.mark.parametrize("name", sorted(PROLOGUES))
def test_prologue_bit_exact(name, golden):
    kind, lam, b, n, M, split, delta = PROLOGUES[name]
    cfg = rt.AssemblyConfig(grid=rt.Grid3(n, rt.Box3(b)), kernel=rt.RadialKernel(kind, lam), M=M,
                            split_index=split, delta=delta)
    ref = rt.reference_for(cfg)
    g = golden[f"prologue_{name}"]
    assert sha(ref.rule.nodes) == g["nodes_sha"]
    assert sha(ref.rule.weights) == g["qweights_sha"]
    assert sha(ref.tensor.weights) == g["weights_sha"]
    assert sha(ref.table) == g["table_sha"]
    assert ref.R == g["R"] and ref.rule.h_M == g["h_M"]
    short, _ = rt.split_tensor(ref, split)
    assert rt.effective_support(short, delta, ref.grid.h) == g["gamma"]
    assert dataclasses.replace(ref, split_index=split).self_value() == g["self_value"]


def test_generators_match_reference(golden):
    g = golden["generators"]
    c1 = rt.generate_random_cluster(64, rt.Box3(6.0), min_sep=1e-9, seed=0, charge_law="uniform")
    assert sha(c1.positions) == g["c1_pos"] and sha(c1.charges) == g["c1_q"]
    c4 = rt.generate_random_cluster(3000, rt.Box3(56.0), 0.8, seed=0, charge_law="uniform")
    assert sha(c4.positions) == g["c4_3000_pos"] and sha(c4.charges) == g["c4_3000_q"]
    lat = rt.generate_lattice((7, 5, 3), 1.25, charge_law="random_sign", seed=3)
    assert sha(lat.positions) == g["lattice_pos"] and sha(lat.charges) == g["lattice_q"]


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_config_systems_and_snap(name, golden):
    g = golden[f"snap_{name}"]
    s = configs.system(name)
    assert sha(s.positions) == g["pos_sha"] and sha(s.charges) == g["q_sha"]
    m = configs.MANIFEST[name]
    snapped = rt.snap_to_grid(s, rt.Grid3(m["n"], rt.Box3(m["b"])))
    assert snapped.count == g["count"] == m["N"]
    assert sha(snapped.indices) == g["indices"]
    assert sha(snapped.base.positions) == g["positions"]
    assert snapped.max_displacement == g["max_disp"]


def test_snap_collision_raises():
    grid = rt.Grid3(8, rt.Box3(1.0))
    sys2 = rt.ParticleSystem(np.array([[0.01, 0.0, 0.0], [-0.01, 0.0, 0.0]]), np.ones(2), rt.Box3(1.0))
    with pytest.raises(rt.ResolutionError):
        rt.snap_to_grid(sys2, grid)


def test_snap_ties_low_and_clip():
    grid = rt.Grid3(8, rt.Box3(1.0))   # h = 0.25
    pos = np.array([[0.125, -0.999, 0.999], [0.0, 0.0, 0.0]])
    s = rt.snap_to_grid(rt.ParticleSystem(pos, np.ones(2), rt.Box3(1.0)), grid)
    assert s.indices[0].tolist() == [4, 1, 7]
    assert s.indices[1].tolist() == [4, 4, 4]


def test_config_validation():
    with pytest.raises(rt.ConfigError):
        rt.ReductionConfig()
    with pytest.raises(rt.ConfigError):
        rt.ReductionConfig(eps=1e-3, ranks=(1, 1, 1))
    with pytest.raises(rt.ConfigError):
        rt.ReductionConfig(ranks=(1, 0, 1))
    with pytest.raises(rt.ConfigError):
        rt.AssemblyConfig(grid=rt.Grid3(8, rt.Box3(1.0)), long_format="dense")
    with pytest.raises(rt.ConfigError):
        rt.AssemblyConfig(grid=rt.Grid3(8, rt.Box3(1.0)), delta=2.0)
    with pytest.raises(rt.DomainError):
        rt.Grid3(7, rt.Box3(1.0))
    with pytest.raises(rt.DomainError):
        rt.ParticleSystem(np.array([[2.0, 0, 0]]), np.ones(1), rt.Box3(1.0))
    with pytest.raises(rt.CapabilityError):
        rt.RadialKernel("coulomb")


def test_particle_file_roundtrip(tmp_path):
    s = configs.system("C1")
    p = tmp_path / "c1.txt"
    rt.save_particles(s, p)
    back = rt.load_particles(p)
    assert np.array_equal(back.positions, s.positions) and np.array_equal(back.charges, s.charges)
    bad = tmp_path / "bad.txt"
    bad.write_text("# rs-particles v1 b=2.0\n0 0 0 1\nnot a number here\n")
    with pytest.raises(rt.ParseError, match="line 3"):
        rt.load_particles(bad)


def test_separation_distance_matches_bruteforce():
    s = rt.generate_random_cluster(5000, rt.Box3(20.0), 0.3, seed=4)
    from scipy.spatial.distance import pdist
    assert rt.separation_distance(s) == float(pdist(s.positions).min())


def test_truncated_spectra_matches_scalar_rule():
    """The vectorised rank rule (critical path after the eigen sync) equals
    the per-mode rule on decaying, flat, zero and forced spectra."""
    import numpy as np
    from paper_1606_09218_b200.rankred import truncated_spectra, truncated_spectrum

    rng = np.random.default_rng(3)
    n, b = 256, 24
    cases = []
    for decay in (0.3, 0.8, 2.0):
        th = np.sort(np.exp(-decay * np.arange(b)) * rng.uniform(0.5, 1.5, b))[::-1]
        cases.append(th)
    cases.append(np.zeros(b))
    thetas = np.stack(cases[:3])
    traces = thetas.sum(axis=1) * (1 + 1e-9)
    for eps in (1e-6, 1e-8, 1e-12):
        for forced in (None, (3, 4, 5)):
            got = truncated_spectra(thetas, traces, n, eps, forced, 200, 2)
            for l in range(3):
                ref = truncated_spectrum(thetas[l], traces[l], n, eps,
                                         None if forced is None else forced[l], 200, 2)
                assert got[l][0] == ref[0]
                assert np.array_equal(got[l][1], ref[1])
                assert np.allclose(got[l][2], ref[2], rtol=0, atol=0)
                assert got[l][3] == ref[3]
    z = truncated_spectra(np.zeros((1, b)), [0.0], n, 1e-6, None, 200, 2)
    assert z[0][0] == truncated_spectrum(np.zeros(b), 0.0, n, 1e-6, None, 200, 2)[0]


def test_rank_rule_fast_matches_scalar_rule():
    import numpy as np
    from paper_1606_09218_b200.rankred import rank_rule_fast, truncated_spectrum

    rng = np.random.default_rng(4)
    n, b = 256, 24
    for trial in range(40):
        decay = rng.uniform(0.2, 3.0)
        th = np.sort(np.exp(-decay * np.arange(b)) * rng.uniform(0.5, 1.5, b))[::-1]
        tr = th.sum() * (1 + rng.uniform(0, 1e-6))
        for eps in (1e-6, 1e-8, 1e-12):
            for forced in (None, (5,)):
                got = rank_rule_fast(th.tolist(), [tr], n, eps, forced, 200, 2)[0]
                ref = truncated_spectrum(th, tr, n, eps, None if forced is None else forced[0],
                                         200, 2)
                assert got[0] == ref[0]
                if ref[0] is not None:
                    assert got[1] == (float(ref[2][ref[0]]) if ref[0] < b else 0.0)
                    assert got[2] == ref[3]


def test_kernels_module_alias():
    """``from rstensor.kernels import ...`` ports by renaming the package."""
    from paper_1606_09218_b200 import kernels, quadrature
    from paper_1606_09218_b200.kernels import (DEFAULT_R_RANGE, QuadratureRule, RadialKernel,  # noqa: F401
                                               ReferenceCanonical, build_quadrature,
                                               effective_support, eval_expansion, project_kernel,
                                               split_rank, split_tensor)
    assert project_kernel is quadrature.project_kernel
    assert kernels.RadialKernel is rt.RadialKernel
