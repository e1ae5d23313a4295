"""SURVEY §8(f) rows 1-2 against the reference's own outputs
(tests/golden/make_golden_next.py): ALS refinement (``c2t_als`` with the
reference default ``max_sweeps=3``) and the canonical long format
(``tucker_to_canonical``)."""
import json
import os

import numpy as np
import pytest

import paper_1606_09218_b200 as rt
from paper_1606_09218_b200 import configs
from oracle import rs_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
META = json.load(open(os.path.join(GOLD, "next.json")))


def setup(name):
    fmt, sweeps = name.split("_")[1], int(name.split("als")[1])
    if name.startswith("tiny"):
        c = orc.small_case(n=32, count=24, seed=5)
        box = rt.Box3(8.0)
        grid, M, split, delta, eps, kind, lam = rt.Grid3(32, box), 15, 7, 1e-6, 1e-8, "newton", 1.0
        system = rt.ParticleSystem(c["positions"], c["charges"], box)
    else:
        m = configs.MANIFEST["C1"]
        box = rt.Box3(m["b"])
        grid, M, split, eps, kind, lam = rt.Grid3(m["n"], box), m["M"], m["split_index"], m["eps"], \
            m["kernel"], m["lam"]
        delta = configs.DELTA if fmt == "tucker" else 1e-4
        system = configs.system("C1")
    cfg = rt.AssemblyConfig(grid=grid, kernel=rt.RadialKernel(kind, lam), M=M, split_index=split,
                            sigma=1.0, delta=delta, long_format=fmt,
                            reduction=rt.ReductionConfig(eps=eps, max_sweeps=sweeps),
                            max_overlap=None, reduce_long=True)
    return system, cfg


@pytest.mark.parametrize("name", ["tiny_tucker_als3", "C1_tucker_als3", "C1_canonical_als0",
                                  "C1_canonical_als3"])
def test_next_rows_match_reference(cuda, name):
    g = META[name]
    z = np.load(os.path.join(GOLD, f"next_{name}.npz"))
    system, cfg = setup(name)
    res = rt.build_rs(system, cfg)
    rep = res.report
    assert rep["tucker_ranks"] == g["report"]["tucker_ranks"]
    if "reduced_canonical_rank" in g["report"]:
        assert rep["reduced_canonical_rank"] == g["report"]["reduced_canonical_rank"]
    n = cfg.grid.n
    grid = rt.dense_rs(res.rs, limit=1 << 40)
    scale = g["grid_max_abs"]
    if "grid" in z:
        err = np.max(np.abs(grid - z["grid"]))
    else:
        s = z["sample_idx"]
        err = np.max(np.abs(grid[s[:, 0], s[:, 1], s[:, 2]] - z["sample_vals"]))
    assert err <= 1e-10 * scale, (name, err / scale)
    vals = rt.eval_rs_many(res.rs, z["eval_idx"])
    assert np.max(np.abs(vals - z["eval_vals"])) <= 1e-12 * scale
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        e = rt.rs_energy(res.rs, res.system, res.reference)
    print(name, "grid", err / scale, "energy", abs(e - g["rs_energy"]) / abs(g["rs_energy"]))
    # three ALS sweeps re-run the reference's SVDs on cuSOLVER with a DMMA
    # matricization: measured 6e-12 relative at C1 (1e-14 without sweeps)
    assert abs(e - g["rs_energy"]) <= (1e-12 if "als0" in name else 2e-11) * abs(g["rs_energy"])
