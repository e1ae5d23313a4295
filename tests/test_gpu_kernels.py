"""Kernel-level checks of librsb200.so against numpy references (float64)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nat(cuda):
    from paper_1606_09218_b200 import _native
    _native.load_library()
    return _native


@pytest.mark.parametrize("n,K", [(8, 2), (37, 130), (64, 64), (256, 700), (130, 4000), (300, 18)])
def test_syrk_matches_numpy(nat, cuda, n, K):
    from paper_1606_09218_b200.rankred import gram
    rng = np.random.default_rng(n + K)
    a = rng.normal(size=(n, K))
    g = gram(cuda.from_numpy(a).cuda()).cpu().numpy()
    ref = a @ a.T
    assert np.allclose(g, ref, rtol=0, atol=1e-13 * np.abs(ref).max() * math.sqrt(K))
    assert np.array_equal(g, g.T)


def test_syrk_deterministic(nat, cuda):
    from paper_1606_09218_b200.rankred import gram
    a = cuda.randn(200, 5000, dtype=cuda.float64, device="cuda")
    g1, g2 = gram(a), gram(a)
    assert cuda.equal(g1, g2)


@pytest.mark.parametrize("M,N,K", [(1, 1, 2), (129, 65, 30), (1000, 256, 712), (77, 300, 8)])
def test_gemm_nt(nat, cuda, M, N, K):
    rng = np.random.default_rng(M * N)
    a = rng.normal(size=(M, K))
    b = rng.normal(size=(N, K))
    A = cuda.from_numpy(a).cuda()
    B = cuda.from_numpy(b).cuda()
    C = cuda.empty((M, N), dtype=cuda.float64, device="cuda")
    nat.check(nat.lib().rs_gemm_nt(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K,
                                   nat.stream_ptr()), "gemm")
    ref = a @ b.T
    assert np.allclose(C.cpu().numpy(), ref, rtol=0, atol=1e-13 * np.abs(ref).max() * math.sqrt(K))


def test_gather_windows(nat, cuda):
    rng = np.random.default_rng(3)
    n, R = 40, 9
    table = rng.normal(size=(2 * n, R))
    starts = np.array([1, 5, 40, 17], dtype=np.int64)
    gs = rng.uniform(1, 2, size=4)
    ts = rng.uniform(1, 2, size=5)
    T = cuda.from_numpy(table).cuda()
    S = cuda.from_numpy(starts).cuda()
    out = cuda.empty((n, 20), dtype=cuda.float64, device="cuda")
    G, Ts = cuda.from_numpy(gs).cuda(), cuda.from_numpy(ts).cuda()  # keep alive across the launch
    nat.check(nat.lib().rs_gather_windows(T.data_ptr(), R, n, S.data_ptr(), 4, 5, 2, G.data_ptr(),
                                          Ts.data_ptr(), out.data_ptr(), 20, nat.stream_ptr()),
              "gather")
    ref = np.concatenate([table[s:s + n, 2:7] * g * ts for s, g in zip(starts, gs)], axis=1)
    assert np.array_equal(out.cpu().numpy(), ref)


def test_snap_bit_exact(nat, cuda):
    import paper_1606_09218_b200 as rt
    from paper_1606_09218_b200 import configs
    for name in ("C2", "C3"):
        s = configs.system(name)
        m = configs.MANIFEST[name]
        grid = rt.Grid3(m["n"], rt.Box3(m["b"]))
        host = rt.snap_to_grid(s, grid)
        dev = rt.snap_device(s.positions, s.charges, s.box, grid)
        assert np.array_equal(dev.indices.cpu().numpy(), host.indices)
        assert np.array_equal(dev.positions.cpu().numpy(), host.base.positions)
        assert dev.max_displacement == host.max_displacement


def test_sum_dd_matches_fsum(nat, cuda):
    from paper_1606_09218_b200.observables import dd_sum
    rng = np.random.default_rng(7)
    v = np.concatenate([rng.normal(size=100000) * 1e8, rng.normal(size=1000), [1e16, -1e16]])
    got = float(dd_sum(cuda.from_numpy(v).cuda()))
    assert got == math.fsum(v)


@pytest.mark.parametrize("n,b", [(256, 64), (96, 32), (512, 96), (32, 32), (256, 24), (100, 24), (512, 32), (1024, 192)])
def test_topeig_graded_spectrum(nat, cuda, n, b):
    """Block subspace iteration + Jacobi vs the known eigensystem of a graded
    PSD matrix (the spectral shape of the RS side-matrix Grams)."""
    from paper_1606_09218_b200.rankred import top_eig
    rng = np.random.default_rng(n + b)
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = 10.0 ** (-np.arange(n) / 2.5)
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    ev, U, tr = top_eig(cuda.from_numpy(np.stack([g, 2 * g])).cuda(), b, iters=3)
    ev, U = ev.cpu().numpy(), U.cpu().numpy()
    keep = int(np.count_nonzero(lam >= 1e-8))
    for m, scale in ((0, 1.0), (1, 2.0)):
        assert np.allclose(ev[m, :keep], scale * lam[:keep], rtol=0, atol=1e-14 * scale)
        proj = np.abs(U[m, :keep] @ q[:, :keep])
        assert np.allclose(np.diag(proj), 1.0, atol=1e-9)
        lead = np.abs(U[m]).argmax(axis=1)
        assert np.all(U[m][np.arange(b), lead] > 0)
    assert np.allclose(tr.cpu().numpy(), [np.trace(g), 2 * np.trace(g)], rtol=1e-14)


def test_shift_hist_deterministic(nat, cuda):
    from paper_1606_09218_b200.rankred import shift_histograms
    rng = np.random.default_rng(1)
    n = 64
    idx = rng.integers(1, n, size=(3000, 3))
    z = rng.normal(size=3000)
    c, cnt = shift_histograms(cuda.from_numpy(idx).cuda(), cuda.from_numpy(z).cuda(), n)
    c = c.cpu().numpy()
    for l in range(3):
        ref = np.zeros(n)
        np.add.at(ref, n - idx[:, l], z * z)
        assert np.allclose(c[l], ref, rtol=1e-14, atol=0)
    assert np.array_equal(cnt.cpu().numpy(), np.bincount(idx[:, 2], minlength=n))


@pytest.mark.parametrize("M,N,K", [(128, 64, 128), (128, 64, 32), (300, 200, 1040), (1, 5, 16),
                                   (1000, 513, 4096)])
def test_tc8_gemm_s8_exact(nat, cuda, M, N, K):
    """tcgen05 kind::i8 GEMM: int32 result bit-exact against numpy int64."""
    rng = np.random.default_rng(M + 7 * N + K)
    a = rng.integers(-128, 128, size=(M, K), dtype=np.int8)
    b = rng.integers(-128, 128, size=(N, K), dtype=np.int8)
    A = cuda.from_numpy(a).cuda()
    B = cuda.from_numpy(b).cuda()
    C = cuda.full((M, N), 7, dtype=cuda.int32, device="cuda")
    nat.check(nat.lib().rs_tc8_gemm_s8(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N,
                                       M, N, K, nat.stream_ptr()), "tc8")
    cuda.cuda.synchronize()
    ref = a.astype(np.int64) @ b.astype(np.int64).T
    got = C.cpu().numpy()
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:5]


@pytest.mark.parametrize("M,N,K,slices", [(128, 64, 64, 7), (300, 200, 1040, 7), (1000, 256, 712, 8),
                                          (77, 130, 32, 6), (513, 70, 3000, 7),
                                          # K <= 160: the A-resident warp-specialised kernel (k_oz_res)
                                          (1000, 256, 132, 7), (40000, 192, 160, 7), (300, 201, 100, 6),
                                          (129, 64, 33, 7)])
def test_oz_gemm_fp64(nat, cuda, M, N, K, slices):
    """Ozaki-split FP64 GEMM on tcgen05 int8 vs numpy fp64: error within the
    split bound K 2^(-7 S) max|A_i.| max|B_j.| (graded magnitudes per row)."""
    rng = np.random.default_rng(M + N + K)
    a = rng.normal(size=(M, K)) * np.exp(rng.uniform(-8, 8, size=(M, 1)))
    b = rng.normal(size=(N, K)) * np.exp(rng.uniform(-8, 8, size=(N, 1)))
    a[:, ::7] *= 1e-6   # mixed magnitudes inside a row
    A = cuda.from_numpy(a).cuda()
    B = cuda.from_numpy(b).cuda()
    C = cuda.empty((M, N), dtype=cuda.float64, device="cuda")
    L = nat.lib()
    ws = cuda.empty(L.rs_oz_workspace_bytes(M, N, K, slices), dtype=cuda.uint8, device="cuda")
    nat.check(L.rs_oz_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 1,
                           slices, 0, ws.data_ptr(), ws.numel(), nat.stream_ptr()), "oz")
    cuda.cuda.synchronize()
    ref = a @ b.T
    scale = np.abs(a).max(1)[:, None] * np.abs(b).max(1)[None, :]
    err = np.abs(C.cpu().numpy() - ref) / scale
    assert err.max() <= 4 * K * 2.0 ** (-7 * slices + 1), err.max()
    # accumulate: C += A B^T on top of the first result
    nat.check(L.rs_oz_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 1,
                           slices, 1, ws.data_ptr(), ws.numel(), nat.stream_ptr()), "oz")
    cuda.cuda.synchronize()
    err = np.abs(C.cpu().numpy() - 2 * ref) / scale
    assert err.max() <= 8 * K * 2.0 ** (-7 * slices + 1), err.max()


@pytest.mark.parametrize("n,b,rank", [(256, 24, 5), (96, 32, 1), (200, 16, 12), (64, 24, 0)])
def test_topeig_rank_deficient(nat, cuda, n, b, rank):
    """Exactly rank-deficient Grams (rank < b): the CGS2 block collapses row
    by row and the restart path (fresh pseudo-random directions) must still
    return an orthonormal Ritz block, the exact nonzero eigenvalues and zeros."""
    from paper_1606_09218_b200.rankred import top_eig
    rng = np.random.default_rng(100 * n + b + rank)
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = np.zeros(n)
    lam[:rank] = 10.0 ** (-np.arange(rank) / 1.5)
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    ev, U, tr = top_eig(cuda.from_numpy(g[None]).cuda(), b, iters=2)
    ev, U = ev.cpu().numpy()[0], U.cpu().numpy()[0]
    assert np.all(np.isfinite(U)) and np.all(np.isfinite(ev))
    assert np.allclose(U @ U.T, np.eye(b), atol=1e-12)          # orthonormal block
    assert np.allclose(ev[:rank], lam[:rank], rtol=0, atol=1e-14)
    assert np.all(np.abs(ev[rank:]) <= 1e-14)
    if rank:
        proj = np.abs(U[:rank] @ q[:, :rank])
        assert np.allclose(np.diag(proj), 1.0, atol=1e-9)


_TUCKER_VARIANT_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_1606_09218_b200 import formats
torch.manual_seed(3)
dev = "cuda"
# r3 in (96, 160] at n >= 256: the Ozaki-split tcgen05 path (k_oz_res) unless RSB200_TUCKER_OZ=0
for n, ranks, lo, hi in [(200, (37, 41, 45), 3, 39), (130, (40, 33, 70), 0, 130), (256, (64, 64, 64), 100, 164),
                         (256, (20, 24, 132), 7, 71), (320, (30, 30, 160), 0, 33), (258, (16, 16, 98), 250, 258)]:
    facs = [torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device=dev))[0].contiguous() for r in ranks]
    core = torch.randn(ranks, dtype=torch.float64, device=dev)
    long = formats.TuckerTensor(core, tuple(facs))
    ref = torch.einsum("abc,ia,jb,kc->ijk", core, facs[0][lo:hi], facs[1], facs[2])
    scale = float(ref.abs().max())
    got = formats.assemble_grid(long, None, lo, hi)                      # ACC = false
    e0 = float((got - ref).abs().max()) / scale
    base = torch.randn_like(ref)
    out = base.clone()
    formats.tucker_accumulate(long, lo, hi, out)                         # ACC = true
    e1 = float((out - base - ref).abs().max()) / scale
    print(n, ranks, e0, e1)
    tol = 1e-13 if ranks[2] <= 96 else 2e-12   # 7 slices of 7 bits: K 2^-49 of the row/column scales
    assert e0 < tol and e1 < tol, (n, ranks, e0, e1)
print("OK")
"""


@pytest.mark.parametrize("res", ["64", "128", "0", "oz0"])
def test_tucker_gemm_variants(cuda, res):
    """A-resident Tucker GEMM (k_tucker_gemm_res, r3 > 32): 64- and 128-row blocks and the
    per-tile plane GEMM (RSB200_TUCKER_RES, read when the library loads -> one process
    each), with and without ACCUMULATE, ragged n, K not a multiple of 16, against einsum
    (formats.py:173-176)."""
    import os
    import subprocess
    import sys
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    env = dict(os.environ)
    if res == "oz0":   # large r3 on the FP64 DMMA kernel as well
        env["RSB200_TUCKER_OZ"] = "0"
    else:
        env["RSB200_TUCKER_RES"] = res
    r = subprocess.run([sys.executable, "-c", _TUCKER_VARIANT_SCRIPT, root], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr


def test_tucker_oz_workspace_fallback(nat, cuda):
    """rs_assemble_planes picks the Ozaki-split Tucker GEMM for 96 < r3 <= 160 only when the
    caller's workspace has room for the slices; a workspace sized for the FP64 path alone
    must still give the Tucker planes (DMMA kernel), not an error (formats.py:173-176)."""
    torch = cuda
    from paper_1606_09218_b200 import formats
    torch.manual_seed(11)
    n, ranks, lo, hi = 256, (16, 16, 100), 10, 18
    facs = [torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda"))[0].contiguous()
            for r in ranks]
    core = torch.randn(ranks, dtype=torch.float64, device="cuda")
    ref = torch.einsum("abc,ia,jb,kc->ijk", core, facs[0][lo:hi], facs[1], facs[2])
    L = nat.lib()
    flags = nat.ASM_LONG
    planes, rmax = hi - lo, max(ranks)
    full = L.rs_assemble_workspace_bytes(n, planes, rmax, 0, 0, flags)
    oz = L.rs_oz_workspace_bytes(planes * n, n, 100, 7)
    small = full - (oz + 255) // 256 * 256
    assert 0 < small < full
    for size in (small, full):
        ws = torch.empty(size, dtype=torch.uint8, device="cuda")
        out = torch.empty((planes, n, n), dtype=torch.float64, device="cuda")
        nat.check(L.rs_assemble_planes(core.data_ptr(), *ranks, facs[0].data_ptr(),
                                       facs[1].data_ptr(), facs[2].data_ptr(), n, None, None, 0,
                                       0, None, None, None, None, None, None, 0, lo, hi, flags,
                                       out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       nat.stream_ptr()), "rs_assemble_planes")
        torch.cuda.synchronize()
        err = float((out - ref).abs().max() / ref.abs().max())
        assert err < 2e-12, (size, err)
