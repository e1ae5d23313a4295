"""The CPU oracle (oracle/rs_oracle.py) pinned against the reference's own outputs."""
import hashlib

import numpy as np
import pytest

from conftest import load_npz
from oracle import rs_oracle as orc
from paper_1606_09218_b200 import configs


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tiny_case(kind):
    c = orc.small_case(n=32, count=24, seed=5, kind=kind)
    return c


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_oracle_prologue_bit_exact(name, golden):
    m = configs.MANIFEST[name]
    p = orc.prologue(m["kernel"], m["lam"], m["b"], m["n"], m["M"], m["split_index"], configs.DELTA)
    g = golden[f"prologue_{name}"]
    assert sha(p["table"]) == g["table_sha"]
    assert sha(p["w"]) == g["weights_sha"]
    assert p["gamma"] == g["gamma"]
    assert orc.self_value(p["table"], p["w"], m["split_index"], p["h"]) == g["self_value"]


@pytest.mark.parametrize("kind", ["newton", "yukawa"])
def test_oracle_tiny_full_pipeline(kind, golden):
    c = tiny_case(kind)
    out = orc.build_and_dense(c)
    g = golden[f"case_tiny_{kind}"]
    z = load_npz(f"case_tiny_{kind}.npz")
    assert list(out["ranks"]) == g["ranks"] and out["gamma"] == g["gamma"]
    ref = z["grid"]
    assert np.max(np.abs(out["grid"] - ref)) <= 1e-13 * np.max(np.abs(ref))
    h = out["h"]
    e = orc.rs_energy(out["core"], out["zs"], out["idx"], c["charges"], out["table"], out["w"],
                      c["split_index"], h)
    assert e == pytest.approx(g["rs_energy"], rel=1e-13)
    e2 = orc.reference_energy(out["idx"], c["charges"], out["table"], out["w"], c["split_index"], h)
    assert e2 == pytest.approx(g["reference_energy"], rel=1e-13)
    for j, f in zip(z["force_idx"], z["forces"]):
        got = orc.force_fd(out["idx"], c["charges"], out["table"], out["w"], c["split_index"], h, j)
        assert np.allclose(got, f, rtol=1e-12, atol=1e-12 * np.abs(z["forces"]).max())
    vals, _ = orc.eval_cct_many(out["ul"], out["wl"], out["gamma"], out["idx"], c["charges"],
                                z["eval_idx"])
    vals = vals + orc.eval_tucker_many(out["core"], out["zs"], z["eval_idx"])
    assert np.allclose(vals, z["eval_vals"], rtol=0, atol=1e-13 * np.abs(z["eval_vals"]).max())


def test_oracle_c1_grid_bit_exact(golden):
    out = orc.build_and_dense(configs.oracle_case("C1"))
    g = golden["case_C1"]
    assert list(out["ranks"]) == g["ranks"]
    assert sha(out["grid"]) == g["grid_sha"]


@pytest.mark.slow
def test_oracle_c2_grid(golden):
    out = orc.build_and_dense(configs.oracle_case("C2"))
    g = golden["case_C2"]
    z = load_npz("case_C2.npz")
    assert list(out["ranks"]) == g["ranks"]
    grid = out["grid"]
    assert np.max(np.abs(grid[128] - z["plane_128"])) <= 1e-13 * g["grid_max_abs"]
    s = z["sample_idx"]
    assert np.max(np.abs(grid[s[:, 0], s[:, 1], s[:, 2]] - z["sample_vals"])) <= 1e-13 * g["grid_max_abs"]


def test_c_dense_cct_matches_numpy_loop():
    rng = np.random.default_rng(0)
    n, g = 24, 5
    L0 = rng.normal(size=(2 * g + 1,) * 3)
    centers = rng.integers(0, n, size=(40, 3))
    z = rng.normal(size=40)
    a = orc.dense_cct_numpy(L0, g, centers, z, n)
    b = orc.dense_cct_c(L0, g, centers, z, n)
    assert np.array_equal(a, b)
    c = orc.dense_cct_c(L0, g, centers, z, n, 7, 13)
    assert np.array_equal(a[7:13], c)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_shift_rhosvd_matches_literal_route(name, golden):
    """The shift-regrouped oracle RHOSVD (used for C3-C5) reproduces the
    reference's literal Gram route: same ranks, same long-part grid."""
    case = configs.oracle_case(name)
    p = orc.prologue(case["kind"], case["lam"], case["b"], case["n"], case["M"],
                     case["split_index"], case["delta"])
    idx, _, _ = orc.snap(case["positions"], case["b"], case["n"])
    core, zs, spectra, ranks = orc.shift_rhosvd(case, p, idx)
    assert list(ranks) == golden[f"case_{name}"]["ranks"]
    z = load_npz(f"case_{name}.npz")
    s = z["sample_idx"][:500]
    vals = orc.eval_tucker_many(core, zs, s)
    ref = z["long_sample"][:500]
    assert np.max(np.abs(vals - ref)) <= 1e-12 * golden[f"case_{name}"]["grid_max_abs"]
    sref = z["spectrum0"]
    keep = sref > 1e-6 * sref[0]          # above the Gram-route rounding floor
    assert np.allclose(spectra[0][:keep.size][keep], sref[keep], rtol=1e-8)
