"""Rank reduction (canonical -> Tucker) on the device.

Reference: ``rankred.py``.  The per-mode spectra come from the Gram route of
``_thin_svd`` (``rankred.py:82-102``): ``G = A A^T`` on FP64 tensor cores
(``rs_syrk``), ``eigh`` (cuSOLVER), descending order, clip at zero, square
root, largest-|entry|-positive signs.  The reference switches to ``gesdd``
for ``K <= 8n``; both routes produce the same left subspace and the same
eps-rank up to rounding, so this package always takes the Gram route and
pins ranks/grids against the reference in ``tests/``.

Two operand forms are supported:

* explicit side matrices (any :class:`CanonicalTensor`, as ``side_svd`` /
  ``rhosvd`` / ``c2t_als`` accept in the reference);
* the shift-structured long part of a particle system (``assemble_long``'s
  columns are windows of one ``(2n, R)`` table), where the Gram is formed
  from the *shift histogram* -- ``G = sum_s c_s sum_k w_k^2 u_k[s:s+n]
  u_k[s:s+n]^T``, ``c_s = sum_{nu: n - j_nu = s} z_nu^2`` -- an exact
  regrouping of ``A A^T`` that shrinks K from ``N R_l`` to ``#shifts * R_l``,
  and the core is projected shift-by-shift (``rs_shift_project`` +
  ``rs_core``) without ever materialising the ``n x N R_l`` side matrices.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import math

import numpy as np

from . import _native as nat
from .errors import ConfigError, DomainError, NumericalError
from .formats import CanonicalTensor, TuckerTensor, is_device, to_device, to_host


@dataclass(frozen=True)
class SvdSpectrum:
    """Per-mode singular values (host, descending) and left vectors (device)."""

    values: tuple
    vectors: tuple

    def __post_init__(self):
        if len(self.values) != 3 or len(self.vectors) != 3:
            raise DomainError("spectrum needs three modes")
        vals = tuple(np.asarray(to_host(s), dtype=np.float64) for s in self.values)
        for s in vals:
            if s.size > 1 and np.any(np.diff(s) > 1e-12 * max(s[0], 1.0)):
                raise DomainError("singular values must be non-increasing")
        object.__setattr__(self, "values", vals)


@dataclass(frozen=True)
class ReductionConfig:
    """``ranks`` xor ``eps`` (tail-energy rule), ALS controls (``rankred.py:43-69``)."""

    ranks: Optional[tuple] = None
    eps: Optional[float] = None
    max_sweeps: int = 3
    eps_c2t: float = 1e-5
    eps_t2c: float = 1e-6

    def __post_init__(self):
        if (self.ranks is None) == (self.eps is None):
            raise ConfigError("set exactly one of ranks and eps")
        if self.ranks is not None:
            object.__setattr__(self, "ranks", tuple(int(r) for r in self.ranks))
            if len(self.ranks) != 3 or min(self.ranks) < 1:
                raise ConfigError(f"ranks must be three positive integers, got {self.ranks}")
        if self.eps is not None and not (0 < self.eps < 1):
            raise ConfigError(f"eps must lie in (0, 1), got {self.eps}")
        if self.max_sweeps < 0:
            raise ConfigError("max_sweeps must be non-negative")


# ------------------------------------------------------------ device pieces
def _pad_even(a):
    """Zero-pad columns to an even count (cp.async 16-byte granularity)."""
    torch = nat._torch()
    if a.shape[1] % 2 == 0 and a.is_contiguous():
        return a
    out = torch.zeros((a.shape[0], a.shape[1] + (a.shape[1] % 2)), dtype=a.dtype, device=a.device)
    out[:, : a.shape[1]] = a
    return out


def gram(a):
    """``a @ a.T`` for a device (n, K) matrix on DMMA (``rs_syrk``)."""
    torch = nat._torch()
    a = _pad_even(a.contiguous())
    n, k = a.shape
    g = torch.empty((n, n), dtype=torch.float64, device=a.device)
    L = nat.lib()
    wsb = L.rs_syrk_workspace_bytes(n, k)
    ws = nat.Workspace.get(wsb, "syrk")
    nat.check(L.rs_syrk(a.data_ptr(), k, n, k, g.data_ptr(), ws.data_ptr(), ws.numel(),
                        nat.stream_ptr()), "rs_syrk")
    return g


def eig_desc(g):
    """Gram eigenpairs in the reference's post-processing (``rankred.py:92-96,
    72-79``): descending, clipped at 0, sqrt, largest-|entry| made positive.
    Returns device (s, z)."""
    torch = nat._torch()
    try:
        vals, vecs = torch.linalg.eigh(g)
    except RuntimeError as exc:  # cuSOLVER failure
        raise NumericalError(f"eigh failed on a {tuple(g.shape)} Gram matrix") from exc
    vals = torch.flip(vals, dims=(-1,)).clamp_min(0.0)
    z = torch.flip(vecs, dims=(-1,))
    return torch.sqrt(vals), fix_signs(z)


def eig_desc_batched(G):
    """Full spectra of a (m, n, n) stack of Grams (``rs_eigh``: one cuSOLVER
    syevd per matrix on forked streams, no host sync), in :func:`eig_desc`'s
    post-processing.  Returns device (values (m, n) descending, clipped at 0,
    not square-rooted; vectors (m, n, n) with the eigenvectors as ROWS,
    largest-|entry| positive)."""
    torch = nat._torch()
    m, n = int(G.shape[0]), int(G.shape[1])
    V = G.contiguous().clone()
    ev = torch.empty((m, n), dtype=torch.float64, device=V.device)
    L = nat.lib()
    wsb = L.rs_eigh_workspace_bytes(m, n)
    if wsb < 0:
        raise NumericalError("rs_eigh: workspace query failed")
    ws = nat.Workspace.get(wsb, "eigh")
    nat.check(L.rs_eigh(V.data_ptr(), m, n, ev.data_ptr(), ws.data_ptr(), ws.numel(),
                        nat.stream_ptr()), "rs_eigh")
    vals = torch.flip(ev, dims=(-1,)).clamp_min(0.0)
    z = fix_signs(torch.flip(V, dims=(-2,)).transpose(-1, -2))   # columns = vectors
    return vals, z.transpose(-1, -2)


def fix_signs(z):
    torch = nat._torch()
    if z.numel() == 0:
        return z
    lead = torch.argmax(torch.abs(z), dim=-2, keepdim=True)
    s = torch.sign(torch.gather(z, -2, lead))
    s = torch.where(s == 0, torch.ones_like(s), s)
    return (z * s).contiguous()


def eps_rank(s: np.ndarray, eps: float) -> int:
    """Smallest r with tail energy sum_{k>=r} s_k^2 <= eps * total (``rankred.py:129-136``)."""
    sq = s * s
    total = float(np.sum(sq))
    if total == 0.0:
        return 1
    tail = np.cumsum(sq[::-1])[::-1]
    ok = np.flatnonzero(tail <= eps * total)
    r = int(ok[0]) if ok.size else s.size
    return max(r, 1)


def select_ranks(mode_sizes, raw_rank: int, values, cfg: ReductionConfig) -> tuple:
    limit = [min(int(n), int(raw_rank)) for n in mode_sizes]
    if cfg.ranks is not None:
        for r, lim in zip(cfg.ranks, limit):
            if r > lim:
                raise ConfigError(f"requested rank {r} exceeds min(n, R) = {lim}")
        return cfg.ranks
    return tuple(min(eps_rank(s, cfg.eps), lim) for s, lim in zip(values, limit))


def core_from_projections(weights, p1, p2, p3):
    """``sum_k xi_k p1[:,k] (x) p2[:,k] (x) p3[:,k]`` (``rankred.py:151-161``) via
    ``rs_core`` with identity shifts (one "particle" per canonical term)."""
    torch = nat._torch()
    w = to_device(weights)
    K = int(w.shape[0])
    r1, r2, r3 = int(p1.shape[0]), int(p2.shape[0]), int(p3.shape[0])
    core = torch.empty((r1, r2, r3), dtype=torch.float64, device="cuda")
    if K == 0:
        return core.zero_()
    ar = torch.arange(K, dtype=torch.int64, device="cuda")
    shift = torch.stack([ar, ar, ar], dim=1).contiguous()
    one = torch.ones(1, dtype=torch.float64, device="cuda")
    L = nat.lib()
    ws = nat.Workspace.get(L.rs_core_workspace_bytes(r1, r2, r3, K, 1), "core")
    pp = [p.contiguous() for p in (p1, p2, p3)]
    nat.check(L.rs_core(pp[0].data_ptr(), pp[1].data_ptr(), pp[2].data_ptr(), r1, r2, r3, K, 1,
                        shift.data_ptr(), w.data_ptr(), one.data_ptr(), K, core.data_ptr(),
                        ws.data_ptr(), ws.numel(), nat.stream_ptr()), "rs_core")
    return core


def _trusted_tucker(core, factors) -> TuckerTensor:
    """Tucker tensor from factors orthonormal by construction (eigenvectors):
    skips the host-synchronising orthonormality probe."""
    t = object.__new__(TuckerTensor)
    object.__setattr__(t, "core", core.contiguous())
    object.__setattr__(t, "factors", tuple(f.contiguous() for f in factors))
    return t


# ------------------------------------------------------- explicit operands
def _thin_svd_dev(a):
    """Left singular pairs by the reference's route (``rankred.py:82-102``):
    Gram + eigh on DMMA for very wide matrices (K > 8n and K > 512), else a
    direct SVD (cuSOLVER) -- the Gram route squares the condition number,
    which the ALS subspaces notice at the 1e-10 level."""
    n, k = int(a.shape[0]), int(a.shape[1])
    if k > 8 * n and k > 512:
        return eig_desc(gram(a))
    torch = nat._torch()
    try:
        u, sv, _ = torch.linalg.svd(a, full_matrices=False)
    except RuntimeError as exc:
        raise NumericalError(f"SVD failed on a {tuple(a.shape)} side matrix") from exc
    return sv, fix_signs(u)


def side_svd(c: CanonicalTensor, weighted: bool = True) -> SvdSpectrum:
    """Per-mode spectra of the (|weight|-scaled) side matrices (``rankred.py:105-126``)."""
    if c.rank == 0:
        raise DomainError("side_svd needs a nonempty tensor")
    w = to_device(c.weights)
    scale = w.abs() if weighted else None
    vals, vecs = [], []
    for u in c.factors:
        ud = to_device(u)
        s, z = _thin_svd_dev(ud * scale if weighted else ud)
        k = min(int(ud.shape[0]), int(ud.shape[1]))
        vals.append(to_host(s)[:k])
        vecs.append(z[:, :k].contiguous())
    return SvdSpectrum(values=tuple(vals), vectors=tuple(vecs))


def _project(factors, c: CanonicalTensor):
    return [f.T @ to_device(u) for f, u in zip(factors, c.factors)]


def rhosvd(c: CanonicalTensor, cfg: ReductionConfig,
           spectrum: Optional[SvdSpectrum] = None) -> TuckerTensor:
    """Reduced HOSVD (``rankred.py:164-177``)."""
    if spectrum is None:
        spectrum = side_svd(c)
    ranks = select_ranks(c.mode_sizes, c.rank, spectrum.values, cfg)
    factors = tuple(to_device(z)[:, :r].contiguous() for z, r in zip(spectrum.vectors, ranks))
    core = core_from_projections(c.weights, *_project(factors, c))
    return TuckerTensor(core=core, factors=factors)


def rhosvd_error_bound(c, spectrum: SvdSpectrum, ranks) -> float:
    """``sum_l sqrt(sum_{k >= r_l} s_{l,k}^2)`` (``rankred.py:180-196``)."""
    total = 0.0
    for s, r in zip(spectrum.values, (int(r) for r in ranks)):
        if r < 0:
            raise DomainError("ranks must be non-negative")
        tail = np.asarray(s)[r:]
        total += float(np.sqrt(np.sum(tail * tail)))
    return total


def _als_matricization(c: CanonicalTensor, projected, mode: int):
    """Mode-``mode`` unfolding of the partially projected tensor
    (``rankred.py:199-215``): one DMMA GEMM ``(U diag(w)) KR^T``."""
    torch = nat._torch()
    others = [m for m in range(3) if m != mode]
    wa, wb = projected[others[0]], projected[others[1]]
    ra, rb = wa.shape[0], wb.shape[0]
    u = to_device(c.factors[mode]) * to_device(c.weights)
    kr = (wa[:, None, :] * wb[None, :, :]).reshape(ra * rb, -1)
    a = _pad_even(u.contiguous())
    b = _pad_even(kr.contiguous())
    out = torch.empty((a.shape[0], ra * rb), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().rs_gemm_nt(a.data_ptr(), a.shape[1], b.data_ptr(), b.shape[1],
                                   out.data_ptr(), ra * rb, a.shape[0], ra * rb, a.shape[1],
                                   nat.stream_ptr()), "rs_gemm_nt")
    return out


def c2t_als(c: CanonicalTensor, cfg: ReductionConfig,
            spectrum: Optional[SvdSpectrum] = None) -> TuckerTensor:
    """RHOSVD start plus up to ``max_sweeps`` ALS sweeps (``rankred.py:218-249``)."""
    if spectrum is None:
        spectrum = side_svd(c)
    ranks = select_ranks(c.mode_sizes, c.rank, spectrum.values, cfg)
    factors = [to_device(z)[:, :r].contiguous() for z, r in zip(spectrum.vectors, ranks)]
    prev_fit = None
    torch = nat._torch()
    for _ in range(cfg.max_sweeps):
        for mode in range(3):
            mat = _als_matricization(c, _project(factors, c), mode)
            _, z = _thin_svd_dev(mat)
            factors[mode] = z[:, : ranks[mode]].contiguous()
        core = core_from_projections(c.weights, *_project(factors, c))
        fit = float(torch.linalg.vector_norm(core))
        if prev_fit is not None and fit - prev_fit <= cfg.eps_c2t * max(fit, 1e-300):
            break
        prev_fit = fit
    core = core_from_projections(c.weights, *_project(factors, c))
    return TuckerTensor(core=core, factors=tuple(factors))


def tucker_to_canonical(t: TuckerTensor, eps_t2c: float = 1e-6) -> CanonicalTensor:
    """Canonical form with rank <= r1 min(r2, r3) (``rankred.py:252-296``);
    the small core SVDs run on the device (cuSOLVER)."""
    torch = nat._torch()
    r1, r2, r3 = t.ranks
    if float(torch.linalg.vector_norm(t.core)) == 0.0:
        return CanonicalTensor.empty(t.mode_sizes)
    u, s, vt = torch.linalg.svd(t.core.reshape(r1, r2 * r3), full_matrices=False)
    s_h = to_host(s)
    keep = eps_rank(s_h, eps_t2c ** 2) if eps_t2c > 0 else int(np.sum(s_h > 0))
    keep = max(min(keep, int(np.sum(s_h > 0))), 1)
    v1, v2, v3 = t.factors
    weights, cols1, cols2, cols3 = [], [], [], []
    for j in range(keep):
        uj, vj = u[:, j], vt[j] * s[j]
        lead = int(torch.argmax(torch.abs(uj)))
        if float(uj[lead]) < 0:
            uj, vj = -uj, -vj
        p, tau, qt = torch.linalg.svd(vj.reshape(r2, r3), full_matrices=False)
        tau_h = to_host(tau)
        for i in range(tau_h.size):
            if tau_h[i] <= 1e-15 * max(tau_h[0], 1e-300):
                break
            pi, qi = p[:, i], qt[i]
            lead = int(torch.argmax(torch.abs(pi)))
            if float(pi[lead]) < 0:
                pi, qi = -pi, -qi
            weights.append(tau[i])
            cols1.append(v1 @ uj)
            cols2.append(v2 @ pi)
            cols3.append(v3 @ qi)
    if not weights:
        return CanonicalTensor.empty(t.mode_sizes)
    return CanonicalTensor(torch.stack(weights), (torch.stack(cols1, 1), torch.stack(cols2, 1),
                                                  torch.stack(cols3, 1)))


# ---------------------------------------------- shift-structured long part
def shift_histograms(idx, z, n: int):
    """(c, cnt3): per-mode shift histograms ``c`` (3, n) -- ``c[l, s] = sum z^2``
    over particles whose mode-l window starts at ``s = n - idx[:, l]`` -- and
    the x3 occupancy counts (n,), one deterministic kernel (``rs_shift_hist``)."""
    torch = nat._torch()
    c = torch.empty((3, n), dtype=torch.float64, device="cuda")
    cnt3 = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib().rs_shift_hist(idx.data_ptr(), z.data_ptr(), int(z.shape[0]), n,
                                      c.data_ptr(), cnt3.data_ptr(), nat.stream_ptr()),
              "rs_shift_hist")
    return c, cnt3


def shifted_grams(table_dev, n: int, w_long_abs, c):
    """Per-mode Grams of the |z w|-weighted long side matrices from the shift
    histograms: ``X_l[:, s R_l + k] = sqrt(c_ls) |w_k| T[s:s+n, k]`` for every
    start s in [0, n) (empty shifts give zero columns), ``G_l = X_l X_l^T`` on
    DMMA -- all three modes in one ``rs_gram_shifted`` call.  Returns (3, n, n)."""
    torch = nat._torch()
    R_l = int(w_long_abs.shape[0])
    G = torch.empty((3, n, n), dtype=torch.float64, device="cuda")
    L = nat.lib()
    ws = nat.Workspace.get(L.rs_gram_shifted_workspace_bytes(n, R_l), "syrk")
    nat.check(L.rs_gram_shifted(table_dev.data_ptr(), table_dev.shape[1], n, R_l, nat.ptr(c),
                                w_long_abs.data_ptr(), G.data_ptr(), ws.data_ptr(), ws.numel(),
                                nat.stream_ptr()), "rs_gram_shifted")
    return G


TOPEIG_BLOCK = 24
TOPEIG_MAX_BLOCK = 96
TOPEIG_WIDE_BLOCK = 192   # eps < 1e-7 on large grids (C5: rank 132)
TOPEIG_ITERS = 2
TOPEIG_SMEM_DOUBLES = 220 * 1024 // 8 - 2


def top_eig_supported(n: int, b: int) -> bool:
    """Block sizes rs_topeig accepts (Jacobi on the b x b Ritz matrix in smem up
    to 96, cuSOLVER on it above)."""
    return (b in (16, 24, 32, 48, 64, 96) or (b % 32 == 0 and 96 < b <= 512)) and b <= n


def top_eig(G, b: int, iters: int = TOPEIG_ITERS):
    """Top-``b`` eigenpairs of a (m, n, n) stack of PSD Grams (``rs_topeig``).
    Returns device (evals (m, b) descending, U (m, b, n) Ritz rows, trace (m,))."""
    torch = nat._torch()
    m, n, _ = G.shape
    evals = torch.empty((m, b), dtype=torch.float64, device="cuda")
    U = torch.empty((m, b, n), dtype=torch.float64, device="cuda")
    tr = torch.empty(m, dtype=torch.float64, device="cuda")
    L = nat.lib()
    ws = nat.Workspace.get(L.rs_topeig_workspace_bytes(m, n, b), "topeig")
    nat.check(L.rs_topeig(G.data_ptr(), m, n, b, iters, evals.data_ptr(), U.data_ptr(),
                          tr.data_ptr(), ws.data_ptr(), ws.numel(), nat.stream_ptr()), "rs_topeig")
    return evals, U, tr


def truncated_spectrum(theta: np.ndarray, trace: float, n: int, eps, forced_rank=None,
                       limit=None, iters: int = TOPEIG_ITERS):
    """Rank rule of ``_eps_rank`` on a top-b spectrum.

    ``theta`` are the b leading Ritz values (clipped at 0); the uncaptured
    remainder ``max(trace - sum theta, 0)`` (rounding noise once b covers the
    numerical rank) joins every tail sum.  Returns (rank or None if b is too
    small to decide / not converged, s values padded to n, tail(r), total).
    """
    theta = np.clip(theta, 0.0, None)
    b = theta.size
    rem = max(float(trace) - float(np.sum(theta)), 0.0) if b < n else 0.0
    total = float(np.sum(theta)) + rem
    tail = np.cumsum(theta[::-1])[::-1] + rem  # tail[r] = sum_{k>=r} lambda_k
    s = np.zeros(n)
    s[:b] = np.sqrt(theta)
    if forced_rank is not None:
        r = int(forced_rank)
    elif total == 0.0:
        r = 1
    else:
        ok = np.flatnonzero(tail <= eps * total)
        if ok.size == 0:
            return None, s, tail, total          # rank >= b: block too small
        r = max(int(ok[0]), 1)
    if limit is not None:
        r = min(r, limit)
    if b < n:
        # Subspace-iteration accuracy of the kept vectors: the angle of the
        # r-th Ritz vector is ~ C (theta_{b-1}/theta_{r-1})^q with C ~ 1e2 for a
        # random start block, and the grid error it causes scales with the
        # tensor mass in that direction, sqrt(theta_{r-1}/theta_0); demand
        # 1e-11 (the grid tolerance is 1e-10).
        if r >= b:
            return None, s, tail, total
        lam_r = theta[r - 1]
        if lam_r <= 0.0 or theta[0] <= 0.0:
            return None, s, tail, total
        if 1e2 * (theta[b - 1] / lam_r) ** iters * np.sqrt(lam_r / theta[0]) > 1e-11:
            return None, s, tail, total
    return r, s, tail, total


def truncated_spectra(thetas: np.ndarray, traces, n: int, eps, forced=None, limit=None,
                      iters: int = TOPEIG_ITERS):
    """:func:`truncated_spectrum` for all modes at once (one vectorised pass
    over the (m, b) Ritz values: this runs on the critical path between the
    eigen block's synchronisation and the core launch).  Returns a list of
    (rank or None, s, tail, total) per mode, identical to the scalar rule."""
    th = np.clip(np.asarray(thetas, dtype=np.float64), 0.0, None)
    m, b = th.shape
    sums = th.sum(axis=1)
    rem = np.maximum(np.asarray(traces, dtype=np.float64) - sums, 0.0) if b < n else np.zeros(m)
    totals = sums + rem
    tails = np.cumsum(th[:, ::-1], axis=1)[:, ::-1] + rem[:, None]
    ok = tails <= eps * totals[:, None]
    first = np.where(ok.any(axis=1), ok.argmax(axis=1), -1)
    out = []
    for l in range(m):
        s = np.zeros(n)
        s[:b] = np.sqrt(th[l])
        tail, total = tails[l], float(totals[l])
        if forced is not None and forced[l] is not None:
            r = int(forced[l])
        elif total == 0.0:
            r = 1
        elif first[l] < 0:
            out.append((None, s, tail, total))
            continue
        else:
            r = max(int(first[l]), 1)
        if limit is not None:
            r = min(r, limit)
        if b < n:
            lam_r = th[l, r - 1] if 0 < r <= b else 0.0
            if (r >= b or lam_r <= 0.0 or th[l, 0] <= 0.0 or
                    1e2 * (th[l, b - 1] / lam_r) ** iters * np.sqrt(lam_r / th[l, 0]) > 1e-11):
                out.append((None, s, tail, total))
                continue
        out.append((r, s, tail, total))
    return out


def rank_rule_fast(thetas, traces, n: int, eps, forced=None, limit=None,
                   iters: int = TOPEIG_ITERS):
    """:func:`truncated_spectra` without the spectra arrays, in plain Python
    floats (a few dozen values per mode; this sits between the eigen block's
    synchronisation and the core launch).  Returns (rank or None, tail at the
    rank, total) per mode."""
    out = []
    m = len(traces)
    b = len(thetas) // m
    for l in range(m):
        th = [x if x > 0.0 else 0.0 for x in thetas[l * b:(l + 1) * b]]
        tot_th = float(np.sum(np.asarray(th)))   # same order as truncated_spectrum
        rem = max(float(traces[l]) - tot_th, 0.0) if b < n else 0.0
        total = tot_th + rem
        tails = [0.0] * b
        acc = 0.0
        for k in range(b - 1, -1, -1):
            acc += th[k]
            tails[k] = acc + rem
        if forced is not None and forced[l] is not None:
            r = int(forced[l])
        elif total == 0.0:
            r = 1
        else:
            thr = eps * total
            r = next((k for k in range(b) if tails[k] <= thr), -1)
            if r < 0:
                out.append((None, 0.0, total))
                continue
            r = max(r, 1)
        if limit is not None:
            r = min(r, limit)
        if b < n:
            lam_r = th[r - 1] if 0 < r <= b else 0.0
            if (r >= b or lam_r <= 0.0 or th[0] <= 0.0 or
                    1e2 * (th[b - 1] / lam_r) ** iters * math.sqrt(lam_r / th[0]) > 1e-11):
                out.append((None, 0.0, total))
                continue
        out.append((r, tails[r] if r < b else 0.0, total))
    return out


def shifted_core(table_dev, n: int, zs, starts, z, w_long):
    """RHOSVD core of the shift-structured long part."""
    torch = nat._torch()
    R_l = int(w_long.shape[0])
    ld = int(table_dev.shape[1])
    L = nat.lib()
    tts = [torch.empty((int(zl.shape[1]), n, R_l), dtype=torch.float64, device="cuda") for zl in zs]
    nat.check(L.rs_shift_project3(zs[0].data_ptr(), zs[1].data_ptr(), zs[2].data_ptr(),
                                  int(zs[0].shape[1]), int(zs[1].shape[1]), int(zs[2].shape[1]), n,
                                  table_dev.data_ptr(), ld, R_l, n, tts[0].data_ptr(),
                                  tts[1].data_ptr(), tts[2].data_ptr(), nat.stream_ptr()),
              "rs_shift_project3")
    r1, r2, r3 = (int(zl.shape[1]) for zl in zs)
    count = int(z.shape[0])
    core = torch.empty((r1, r2, r3), dtype=torch.float64, device="cuda")
    ws = nat.Workspace.get(L.rs_core_workspace_bytes(r1, r2, r3, count, R_l), "core")
    nat.check(L.rs_core(tts[0].data_ptr(), tts[1].data_ptr(), tts[2].data_ptr(), r1, r2, r3, n,
                        R_l, starts.data_ptr(), z.data_ptr(), w_long.data_ptr(), count,
                        core.data_ptr(), ws.data_ptr(), ws.numel(), nat.stream_ptr()), "rs_core")
    return core
