"""The fused tensor-core short-range kernel (rs_assemble_short_mma,
RS_SHORT_MMA) against the plane-GEMM path, the reference's golden grids and
the oracle's C dense_cct (formats.py:423-445).

The kernel never materialises an operand: A fragments are outer products of
shared-memory staged 1-D factors summed over the candidate copies, B
fragments are gathered from the same table.  It must agree with the other
device paths to rounding and stay within BASELINE's 1e-10 of the reference.
"""
import numpy as np
import pytest

import paper_1606_09218_b200 as rt
from conftest import load_npz
from oracle import rs_oracle as orc
from paper_1606_09218_b200 import _native as nat
from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.formats import assemble_grid
from test_gpu_parity import case_inputs
from test_gpu_short_l0 import small

pytestmark = pytest.mark.gpu

GRID_TOL = 1e-10
AGREE_TOL = 1e-12


def methods(res, monkeypatch, names=("gemm", "mma"), **kw):
    out = {}
    for m in names:
        monkeypatch.setenv("RSB200_SHORT", m)
        out[m] = assemble_grid(res.rs.long, res.rs.short, **kw).cpu().numpy()
    monkeypatch.delenv("RSB200_SHORT")
    return [out[m] for m in names]


def test_supported_and_override(monkeypatch):
    L = nat.lib()
    assert L.rs_short_mma_supported(2048, 80, 20) == 1
    assert L.rs_short_mma_supported(1024, 107, 18) == 1
    assert L.rs_short_mma_supported(256, 94, 14) == 1
    assert L.rs_short_mma_supported(4096, 3000, 20) == 0     # table does not fit shared memory
    assert L.rs_short_mma_supported(256, 94, 25) == 0
    monkeypatch.setenv("RSB200_SHORT", "mma")
    assert L.rs_short_method(256, 1000, 94, 14) == nat.SHORT_MMA
    assert L.rs_short_method(2048, 31130, 80, 20) == nat.SHORT_MMA


@pytest.mark.parametrize("build", ["0", "1"])
@pytest.mark.parametrize("name", ["tiny_newton", "tiny_yukawa", "C1", "C2"])
def test_mma_grid_vs_reference(name, build, cuda, golden, monkeypatch):
    monkeypatch.setenv("RSB200_MMA_BUILD", build)
    system, cfg, _ = case_inputs(name)
    res = rt.build_rs(system, cfg)
    gg, gm = methods(res, monkeypatch)
    scale = golden[f"case_{name}"]["grid_max_abs"]
    assert np.max(np.abs(gg - gm)) <= AGREE_TOL * scale
    z = load_npz(f"case_{name}.npz")
    s = z["sample_idx"]
    assert np.max(np.abs(gm[s[:, 0], s[:, 1], s[:, 2]] - z["sample_vals"])) <= GRID_TOL * scale
    if "grid" in z:
        assert np.max(np.abs(gm - z["grid"])) <= GRID_TOL * scale


@pytest.mark.parametrize("build", ["0", "1"])
@pytest.mark.parametrize("n,count,seed,kind", [(50, 40, 3, "newton"), (34, 7, 11, "yukawa"),
                                               (130, 300, 2, "newton"), (32, 1, 4, "newton")])
def test_mma_ragged_sizes_vs_oracle(n, count, seed, kind, build, cuda, monkeypatch):
    """n not a multiple of the 8 x 16 x 64 tile; windows clipped at every face;
    both A-fragment variants (per-lane outer products / DMMA builder)."""
    monkeypatch.setenv("RSB200_MMA_BUILD", build)
    system, cfg, c = small(n, count, seed, kind)
    res = rt.build_rs(system, cfg)
    gg, gm = methods(res, monkeypatch)
    ranks = tuple(int(r) for r in res.report["tucker_ranks"])
    ref = orc.build_and_dense(c, ranks=ranks)["grid"]
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(gm - ref)) <= GRID_TOL * scale
    assert np.max(np.abs(gg - gm)) <= AGREE_TOL * scale


def test_mma_short_only_vs_c_oracle(cuda, monkeypatch):
    """The short part alone (no Tucker planes) against the C dense_cct loop."""
    torch = cuda
    system, cfg, c = case_inputs("C2")
    res = rt.build_rs(system, cfg)
    p = orc.prologue(c["kind"], c["lam"], c["b"], c["n"], c["M"], c["split_index"], c["delta"])
    idx, _, _ = orc.snap(c["positions"], c["b"], c["n"])
    ul, wl = orc.local_window(p["table"], p["w"], c["split_index"], p["gamma"])
    ref = orc.dense_cct_c(orc.local_dense(ul, wl), p["gamma"], idx, c["charges"], c["n"], 60, 140)
    monkeypatch.setenv("RSB200_SHORT", "mma")
    got = assemble_grid(None, res.rs.short, x1_lo=60, x1_hi=140).cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_mma_slab_and_accumulate(cuda, monkeypatch):
    torch = cuda
    system, cfg, _ = case_inputs("C2")
    res = rt.build_rs(system, cfg)
    n = cfg.grid.n
    monkeypatch.setenv("RSB200_SHORT", "mma")
    full = assemble_grid(res.rs.long, res.rs.short)
    slab = assemble_grid(res.rs.long, res.rs.short, x1_lo=37, x1_hi=101)
    assert torch.equal(slab, full[37:101])          # tiles differ, sums do not
    base = torch.full((64, n, n), 0.25, dtype=torch.float64, device="cuda")
    acc = assemble_grid(None, res.rs.short, x1_lo=37, x1_hi=101, out=base.clone(), accumulate=True)
    short = assemble_grid(None, res.rs.short, x1_lo=37, x1_hi=101)
    assert torch.allclose(acc, short + 0.25, rtol=0, atol=1e-13 * (0.25 + float(short.abs().max())))
    again = assemble_grid(None, res.rs.short, x1_lo=37, x1_hi=101)
    assert torch.equal(short, again)                # deterministic under dynamic tile scheduling


def test_mma_prefetch_matches(cuda, golden, monkeypatch):
    """build_rs(prefetch_dense=True): rs_front launches the fused kernel on the
    side stream when the method says so."""
    system, cfg, _ = case_inputs("C2")
    monkeypatch.setenv("RSB200_SHORT", "mma")
    res = rt.build_rs(system, cfg, prefetch_dense=True)
    grid = rt.dense_rs(res.rs, limit=1 << 40, device=True).cpu().numpy()
    res5 = rt.build_rs(system, cfg, prefetch_dense=(10, 200), prefetch_groups=5)
    part = rt.dense_rs(res5.rs, limit=1 << 40, x1_range=(10, 200))
    monkeypatch.setenv("RSB200_SHORT", "gemm")
    ref = assemble_grid(res.rs.long, res.rs.short).cpu().numpy()
    scale = golden["case_C2"]["grid_max_abs"]
    assert np.max(np.abs(grid - ref)) <= AGREE_TOL * scale
    assert np.max(np.abs(part - ref[10:200])) <= AGREE_TOL * scale


@pytest.mark.slow
@pytest.mark.parametrize("name,planes", [("C3", (1, 200, 256, 511)), ("C4", (1, 511, 700, 1023)),
                                         ("C5", (1, 1023, 1500, 2047))])
def test_mma_large_planes_vs_c_oracle(name, planes, cuda, monkeypatch):
    """Full-size configs: x1 planes of the short part against the C dense_cct."""
    c = configs.oracle_case(name)
    res = rt.build_rs(configs.system(name), configs.assembly_config(name))
    p = orc.prologue(c["kind"], c["lam"], c["b"], c["n"], c["M"], c["split_index"], c["delta"])
    idx, _, _ = orc.snap(c["positions"], c["b"], c["n"])
    ul, wl = orc.local_window(p["table"], p["w"], c["split_index"], p["gamma"])
    L0 = orc.local_dense(ul, wl)
    monkeypatch.setenv("RSB200_SHORT", "mma")
    pairs = []
    for x in planes:
        ref = orc.dense_cct_c(L0, p["gamma"], idx, c["charges"], c["n"], x, x + 1)[0]
        got = assemble_grid(None, res.rs.short, x1_lo=x, x1_hi=x + 1).cpu().numpy()[0]
        pairs.append((x, got, ref))
    scale = max(float(np.max(np.abs(r))) for _, _, r in pairs)
    for x, got, ref in pairs:
        assert np.max(np.abs(got - ref)) <= 1e-12 * scale, (name, x)
