"""The low-overlap short-range path (dense-L0 gather, rs_assemble_short_l0)
against the plane-GEMM path, the reference's golden grids and the oracle.

Both methods evaluate dense_cct (formats.py:423-445); the gather reads the
dense local tensor L0 = local.dense() (formats.py:432) exactly as the
reference does, so the two device paths agree to rounding (1e-12 of max|P|)
and each stays within the BASELINE grid tolerance (1e-10) of the reference.
"""
import numpy as np
import pytest

import paper_1606_09218_b200 as rt
from conftest import load_npz
from oracle import rs_oracle as orc
from paper_1606_09218_b200 import _native as nat
from paper_1606_09218_b200.formats import assemble_grid
from test_gpu_parity import case_inputs

pytestmark = pytest.mark.gpu

GRID_TOL = 1e-10
AGREE_TOL = 1e-12


def small(n, count, seed, kind="newton"):
    c = orc.small_case(n=n, count=count, seed=seed, kind=kind)
    box = rt.Box3(c["b"])
    cfg = rt.AssemblyConfig(grid=rt.Grid3(n, box),
                            kernel=rt.RadialKernel(kind, c["lam"] if kind == "yukawa" else 1.0),
                            M=c["M"], split_index=c["split_index"], sigma=1.0, delta=c["delta"],
                            long_format="tucker",
                            reduction=rt.ReductionConfig(eps=c["eps"], max_sweeps=0),
                            max_overlap=None)
    return rt.ParticleSystem(c["positions"], c["charges"], box), cfg, c


def both(res, monkeypatch, **kw):
    out = {}
    for m in ("gemm", "l0"):
        monkeypatch.setenv("RSB200_SHORT", m)
        out[m] = assemble_grid(res.rs.long, res.rs.short, **kw).cpu().numpy()
    monkeypatch.delenv("RSB200_SHORT")
    return out["gemm"], out["l0"]


def test_method_choice_and_override(monkeypatch):
    L = nat.lib()
    monkeypatch.delenv("RSB200_SHORT", raising=False)
    # default: the fused tensor-core kernel wherever its table fits shared memory
    assert L.rs_short_method(2048, 31130, 80, 20) == nat.SHORT_MMA
    assert L.rs_short_method(256, 1000, 94, 14) == nat.SHORT_MMA
    assert L.rs_short_method(1024, 100000, 107, 18) == nat.SHORT_MMA
    # beyond it: the L0 gather at low overlap (15 copies / point), else the plane GEMM
    assert L.rs_short_method(4096, 31130, 700, 20) == nat.SHORT_GEMM   # pair table too wide too
    assert L.rs_short_method(4096, 100, 120, 30) == nat.SHORT_L0       # Rs beyond the fused kernel
    monkeypatch.setenv("RSB200_SHORT", "l0")
    assert L.rs_short_method(256, 1000, 94, 14) == nat.SHORT_L0
    monkeypatch.setenv("RSB200_SHORT", "gemm")
    assert L.rs_short_method(2048, 31130, 80, 20) == nat.SHORT_GEMM


def test_l0_table_vs_oracle(cuda):
    system, cfg, _ = case_inputs("C2")
    res = rt.build_rs(system, cfg)
    sh = res.rs.short
    P = sh.l0_table().cpu().numpy()
    ul = np.asarray(sh.local.factors[0])
    ref = orc.local_dense(ul, np.asarray(sh.local.weights))
    # unfold the pair table: L0[a, b, c] = P[par, |a-g|, b, c + 2 - par]
    g = sh.gamma
    w = 2 * g + 1
    fa = np.abs(np.arange(w) - g)
    for par in (0, 1):
        l0 = P[par][fa][:, :, 2 - par:2 - par + w]
        assert l0.shape == ref.shape
        assert np.max(np.abs(l0 - ref)) <= 1e-14 * np.max(np.abs(ref))
    # zero margins: a 16-byte pair straddling the window edge reads zeros
    assert not P[0][..., :2].any() and not P[0][..., 2 + w:].any()
    assert not P[1][..., :1].any() and not P[1][..., 1 + w:].any()


@pytest.mark.parametrize("name", ["tiny_newton", "tiny_yukawa", "C1", "C2"])
def test_l0_grid_vs_reference(name, cuda, golden, monkeypatch):
    system, cfg, _ = case_inputs(name)
    res = rt.build_rs(system, cfg)
    gg, gl = both(res, monkeypatch)
    scale = golden[f"case_{name}"]["grid_max_abs"]
    assert np.max(np.abs(gg - gl)) <= AGREE_TOL * scale
    z = load_npz(f"case_{name}.npz")
    s = z["sample_idx"]
    assert np.max(np.abs(gl[s[:, 0], s[:, 1], s[:, 2]] - z["sample_vals"])) <= GRID_TOL * scale
    if "grid" in z:
        assert np.max(np.abs(gl - z["grid"])) <= GRID_TOL * scale


@pytest.mark.parametrize("n,count,seed,kind", [(50, 40, 3, "newton"), (34, 7, 11, "yukawa"),
                                               (130, 300, 2, "newton")])
def test_l0_ragged_sizes_vs_oracle(n, count, seed, kind, cuda, monkeypatch):
    """n not a multiple of the 8 x 16 x 128 tile; windows clipped at every face."""
    system, cfg, c = small(n, count, seed, kind)
    res = rt.build_rs(system, cfg)
    gg, gl = both(res, monkeypatch)
    ranks = tuple(int(r) for r in res.report["tucker_ranks"])
    ref = orc.build_and_dense(c, ranks=ranks)["grid"]
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(gl - ref)) <= GRID_TOL * scale
    assert np.max(np.abs(gg - gl)) <= AGREE_TOL * scale


def test_l0_slab_and_accumulate(cuda, monkeypatch):
    torch = cuda
    system, cfg, _ = case_inputs("C2")
    res = rt.build_rs(system, cfg)
    n = cfg.grid.n
    monkeypatch.setenv("RSB200_SHORT", "l0")
    full = assemble_grid(res.rs.long, res.rs.short)
    slab = assemble_grid(res.rs.long, res.rs.short, x1_lo=37, x1_hi=101)
    assert torch.equal(slab, full[37:101])
    # short only, accumulated onto an existing slab
    base = torch.full((64, n, n), 0.25, dtype=torch.float64, device="cuda")
    acc = assemble_grid(None, res.rs.short, x1_lo=37, x1_hi=101, out=base.clone(), accumulate=True)
    short = assemble_grid(None, res.rs.short, x1_lo=37, x1_hi=101)
    assert torch.allclose(acc, short + 0.25, rtol=0, atol=1e-13 * (0.25 + float(short.abs().max())))


def test_l0_prefetch_matches(cuda, golden, monkeypatch):
    """build_rs(prefetch_dense=True): the short planes come from rs_front's
    side-stream launch (gather when RSB200_SHORT=l0)."""
    system, cfg, _ = case_inputs("C2")
    monkeypatch.setenv("RSB200_SHORT", "l0")
    res = rt.build_rs(system, cfg, prefetch_dense=True)
    grid = rt.dense_rs(res.rs, limit=1 << 40, device=True).cpu().numpy()
    monkeypatch.setenv("RSB200_SHORT", "gemm")
    ref = assemble_grid(res.rs.long, res.rs.short).cpu().numpy()
    scale = golden["case_C2"]["grid_max_abs"]
    assert np.max(np.abs(grid - ref)) <= AGREE_TOL * scale


@pytest.mark.parametrize("method", ["gemm", "l0"])
@pytest.mark.parametrize("rng_", [None, (37, 101)])
def test_grouped_prefetch_to_host(method, rng_, cuda, golden, monkeypatch):
    """build_rs(prefetch_groups=k): rs_front finishes the short planes group by
    group, build_rs adds the Tucker part per group, dense_rs copies each group
    to the host as soon as it is final -- same grid as the one-shot path."""
    system, cfg, _ = case_inputs("C2")
    monkeypatch.setenv("RSB200_SHORT", method)
    n = cfg.grid.n
    lo, hi = (0, n) if rng_ is None else rng_
    pre = True if rng_ is None else rng_
    ref = assemble_grid(rt.build_rs(system, cfg).rs.long, None, lo, hi)
    res = rt.build_rs(system, cfg, prefetch_dense=pre, prefetch_groups=5)
    host = rt.dense_rs(res.rs, limit=1 << 40, x1_range=None if rng_ is None else rng_)
    full = assemble_grid(res.rs.long, res.rs.short, lo, hi).cpu().numpy()
    scale = golden["case_C2"]["grid_max_abs"]
    assert host.shape == ((n, n, n) if rng_ is None else (hi - lo, n, n))
    assert np.max(np.abs(host.reshape(full.shape) - full)) <= AGREE_TOL * scale
    assert ref.shape[0] == hi - lo


def test_prefetch_into_caller_buffer(cuda, golden):
    """build_rs(prefetch_out=buf): the grid lands in the caller's buffer."""
    torch = cuda
    system, cfg, _ = case_inputs("C2")
    n = cfg.grid.n
    buf = torch.full((n, n, n), float("nan"), dtype=torch.float64, device="cuda")
    res = rt.build_rs(system, cfg, prefetch_dense=True, prefetch_out=buf)
    grid = rt.dense_rs(res.rs, limit=1 << 40, device=True)
    assert grid.data_ptr() == buf.data_ptr()
    ref = assemble_grid(res.rs.long, res.rs.short)
    scale = golden["case_C2"]["grid_max_abs"]
    assert float((grid - ref).abs().max()) <= AGREE_TOL * scale
    with pytest.raises(rt.DomainError):
        rt.build_rs(system, cfg, prefetch_dense=True, prefetch_out=buf[:10])
