"""CPU ORACLE for the RS assembly path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module.  It is the checker, never the
product: the package ``paper_1606_09218_b200`` does not import it.

It restates the reference algorithm (``rstensor`` 0.1.0 at /root/reference,
pure numpy/scipy) with plain arrays, function by function, citing the
reference file:line it follows.  Parity is pinned two ways:

* ``tests/golden/*.npz`` were produced by running the reference itself
  (``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks
  this module against them (bit-exact for the host prologue, 1e-13 for grids);
* the hot loop of ``dense_cct`` (``formats.py:432-445``) also has a C
  restatement (``oracle/dense_cct.c``, OpenMP) so full-size grids finish in
  seconds; it is checked against the numpy loop here.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
from scipy.special import erf

SQRT_PI = math.sqrt(math.pi)
_HERE = os.path.dirname(os.path.abspath(__file__))


# ------------------------------------------------ particles.py:62-99, 302-329
def grid_h(b: float, n: int) -> float:
    return 2.0 * b / n


def snap(positions: np.ndarray, b: float, n: int):
    """Nearest node, ties low, clipped to [1, n-1] (particles.py:311-318)."""
    h = grid_h(b, n)
    fi = positions / h + n // 2
    idx = np.clip(np.ceil(fi - 0.5).astype(np.int64), 1, n - 1)
    snapped = (idx.astype(np.float64) - n // 2) * h
    disp = np.linalg.norm(positions - snapped, axis=1)
    keys = np.unique(idx, axis=0)
    if keys.shape[0] != idx.shape[0]:
        raise ValueError("collision")
    return idx, snapped, float(disp.max())


# ------------------------------------------------------- kernels.py:125-283
def _gsum(t, a, r):
    return (a[None, :] * np.exp(-np.outer(r * r, t * t))).sum(axis=1)


def _newton(M, h, alpha):
    u = np.arange(M + 1) * h
    t = alpha * np.sinh(u)
    a = (2.0 / SQRT_PI) * alpha * np.cosh(u) * h
    a[0] *= 0.5
    return t, a


def _golden_min(f, lo, hi, iters):
    g = (math.sqrt(5.0) - 1.0) / 2.0
    c, d = hi - g * (hi - lo), lo + g * (hi - lo)
    fc, fd = f(c), f(d)
    for _ in range(iters):
        if fc < fd:
            hi, d, fd = d, c, fc
            c = hi - g * (hi - lo)
            fc = f(c)
        else:
            lo, c, fc = c, d, fd
            d = lo + g * (hi - lo)
            fd = f(d)
    return lo, hi


def _density(kind, lam, t):
    if kind == "newton":
        return np.full_like(t, 2.0 / SQRT_PI)
    safe = np.where(t > 0, t, 1.0)
    damp = np.where(t > 0, np.exp(-lam * lam / (4.0 * safe * safe)), 0.0)
    if kind == "yukawa":
        return (2.0 / SQRT_PI) * damp
    return (lam / SQRT_PI) * damp / np.where(t > 0, safe * safe, 1.0)


def _geometric(kind, lam, M, t_lo, t_hi):
    v = np.linspace(math.log(t_lo), math.log(t_hi), M)
    t = np.exp(v)
    hv = v[1] - v[0] if M > 1 else 1.0
    a = _density(kind, lam, t) * t * hv
    if M > 1:
        a[0] *= 0.5
        a[-1] *= 0.5
    return np.concatenate([[0.0], t]), np.concatenate([[0.0], a])


def kernel_values(kind, lam, r):
    if kind == "newton":
        return 1.0 / r
    if kind == "yukawa":
        return np.exp(-lam * r) / r
    if kind == "slater":
        return np.exp(-lam * r)
    return np.exp(-lam * r * r)


def quadrature(kind: str, lam: float, M: int, C0: float, r_lo: float, r_hi: float):
    """Nodes/weights of build_quadrature (kernels.py:241-283)."""
    h = C0 * math.log(max(M, 2)) / M
    probes = np.geomspace(r_lo, r_hi, 128)
    if kind == "newton":
        target = 1.0 / probes

        def err(la):
            t, a = _newton(M, h, math.exp(la))
            return float(np.max(np.abs(_gsum(t, a, probes) - target) / target))

        lo, hi = _golden_min(err, math.log(1e-6), math.log(10.0), 72)
        return _newton(M, h, math.exp(0.5 * (lo + hi)))
    target = kernel_values(kind, lam, probes)

    def err2(x):
        t, a = _geometric(kind, lam, M, math.exp(x[0]), math.exp(x[1]))
        return float(np.max(np.abs(_gsum(t, a, probes) - target) / np.abs(target)))

    x = [math.log(max(math.sqrt(lam / (2.0 * r_hi)) / 4.0, 1e-4)),
         math.log(math.sqrt(math.log(1e8)) / r_lo)]
    init = [(x[0] - 5.0, x[0] + 5.0), (x[1] - 5.0, x[1] + 5.0)]
    for _ in range(6):
        for dim in (0, 1):
            def f(v, dim=dim):
                y = list(x)
                y[dim] = v
                return err2(y)
            lo, hi = _golden_min(f, init[dim][0], init[dim][1], 40)
            x[dim] = 0.5 * (lo + hi)
    return _geometric(kind, lam, M, math.exp(x[0]), math.exp(x[1]))


def doubled_table(t, a, b: float, n: int):
    """(2n, R) unit columns + weights a |col|^3 (kernels.py:358-398, doubled grid)."""
    n2 = 2 * n
    h = 2.0 * (2.0 * b) / n2
    x = (np.arange(n2) - n2 // 2) * h
    cols = np.empty((n2, t.size))
    for k, tk in enumerate(t):
        cols[:, k] = h if tk == 0.0 else (SQRT_PI / (2.0 * tk)) * (
            erf(tk * (x + 0.5 * h)) - erf(tk * (x - 0.5 * h)))
    norms = np.linalg.norm(cols, axis=0)
    unit = cols / np.where(norms > 0, norms, 1.0)
    return np.ascontiguousarray(unit), a * norms ** 3


def gamma_of(table, w, split_index, delta, h):
    """effective_support on the short terms (kernels.py:457-482)."""
    u = table[:, split_index + 1:]
    ws = w[split_index + 1:]
    n2 = u.shape[0]
    c = n2 // 2
    d = np.arange(1, n2 - c)
    g = 0
    for k in range(u.shape[1]):
        peak = float(u[c, k])
        scale = ws[k] * peak * peak / h ** 3
        above = np.nonzero(scale * np.maximum(u[c + d, k], u[c - d, k]) > delta)[0]
        if above.size:
            g = max(g, int(d[above[-1]]))
    return g


def local_window(table, w, split_index, gamma):
    """assemble_short local tensor: short window, normalised (assembly.py:160-165,
    formats.py:80-91); returns (ul (W, R_s), wl (R_s,))."""
    c = table.shape[0] // 2
    u = table[c - gamma:c + gamma + 1, split_index + 1:]
    wl = w[split_index + 1:].copy()
    norms = np.linalg.norm(u, axis=0)
    safe = np.where(norms > 0, norms, 1.0)
    for _ in range(3):
        wl = wl * norms
    return np.ascontiguousarray(u / safe), wl


# --------------------------------------------- assembly.py:111-136, rankred.py
def long_side_matrices(table, w, idx, z, split_index):
    n = table.shape[0] // 2
    nt = split_index + 1
    weights = (z[:, None] * w[None, :nt]).reshape(-1)
    facs = []
    for l in range(3):
        out = np.empty((n, idx.shape[0] * nt))
        st = n - idx[:, l]
        for nu in range(idx.shape[0]):
            out[:, nu * nt:(nu + 1) * nt] = table[st[nu]:st[nu] + n, :nt]
        facs.append(out)
    return weights, facs


def thin_svd(a):
    """rankred.py:82-102 (Gram route for K > 8n and K > 512, else gesdd)."""
    n, r = a.shape
    if r > 8 * n and r > 512:
        vals, vecs = np.linalg.eigh(a @ a.T)
        order = np.argsort(vals)[::-1]
        vals = np.clip(vals[order], 0.0, None)
        z, s = vecs[:, order], np.sqrt(vals)
    else:
        z, s, _ = np.linalg.svd(a, full_matrices=False)
    lead = np.abs(z).argmax(axis=0)
    sg = np.sign(z[lead, np.arange(z.shape[1])])
    sg[sg == 0] = 1.0
    return z * sg, s


def eps_rank(s, eps):
    total = float(np.sum(s * s))
    if total == 0.0:
        return 1
    tail = np.cumsum((s * s)[::-1])[::-1]
    ok = np.nonzero(tail <= eps * total)[0]
    return max(int(ok[0]) if ok.size else s.size, 1)


def rhosvd(weights, facs, eps=None, ranks=None):
    """side_svd(weighted) + c2t_als(max_sweeps=0) (rankred.py:105-126, 218-249)."""
    spec = [thin_svd(u * np.abs(weights)) for u in facs]
    if ranks is None:
        ranks = tuple(min(eps_rank(s, eps), min(u.shape)) for (z, s), u in zip(spec, facs))
    zs = [z[:, :r] for (z, _), r in zip(spec, ranks)]
    pr = [zz.T @ u for zz, u in zip(zs, facs)]
    core = np.zeros(tuple(ranks))
    for lo in range(0, weights.size, 2048):
        hi = min(lo + 2048, weights.size)
        core += np.einsum("k,ak,bk,ck->abc", weights[lo:hi], pr[0][:, lo:hi], pr[1][:, lo:hi],
                          pr[2][:, lo:hi], optimize=True)
    return core, zs, [s for _, s in spec], tuple(ranks)


# ------------------------------------------------------ formats.py:173-453
def tucker_dense(core, zs, x1=slice(None)):
    return np.einsum("abc,ia,jb,lc->ijl", core, zs[0][x1], zs[1], zs[2], optimize=True)


def local_dense(ul, wl):
    return np.einsum("k,ik,jk,lk->ijl", wl, ul, ul, ul, optimize=True)


def dense_cct_numpy(L0, gamma, centers, z, n):
    """The reference loop (formats.py:440-444), window clipped at the faces."""
    out = np.zeros((n, n, n))
    for nu in range(centers.shape[0]):
        c = centers[nu]
        lo = np.maximum(c - gamma, 0)
        hi = np.minimum(c + gamma, n - 1)
        llo = lo - (c - gamma)
        lhi = hi - (c - gamma)
        out[lo[0]:hi[0] + 1, lo[1]:hi[1] + 1, lo[2]:hi[2] + 1] += z[nu] * L0[
            llo[0]:lhi[0] + 1, llo[1]:lhi[1] + 1, llo[2]:lhi[2] + 1]
    return out


_clib = None


def _c_oracle():
    global _clib
    if _clib is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        lib.oracle_dense_cct.restype = None
        lib.oracle_dense_cct.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        _clib = lib
    return _clib


def dense_cct_c(L0, gamma, centers, z, n, x1_lo=0, x1_hi=None):
    """Same sum as dense_cct_numpy, x1 planes [x1_lo, x1_hi), OpenMP C loop
    (particle order per plane is the reference's, so results are identical)."""
    x1_hi = n if x1_hi is None else x1_hi
    L0 = np.ascontiguousarray(L0, dtype=np.float64)
    c = np.ascontiguousarray(centers, dtype=np.int64)
    zz = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros((x1_hi - x1_lo, n, n))
    _c_oracle().oracle_dense_cct(L0.ctypes.data, gamma, c.ctypes.data, zz.ctypes.data,
                                 c.shape[0], n, x1_lo, x1_hi, out.ctypes.data)
    return out


# -------------------------------------------------- formats.py:340-420
def eval_tucker_many(core, zs, idx):
    tmp = np.tensordot(zs[0][idx[:, 0]], core, axes=(1, 0))
    tmp = np.einsum("mbc,mb->mc", tmp, zs[1][idx[:, 1]])
    return np.einsum("mc,mc->m", tmp, zs[2][idx[:, 2]])


def eval_cct_many(ul, wl, gamma, centers, z, idx):
    out = np.empty(idx.shape[0])
    hits = np.empty(idx.shape[0], dtype=np.int64)
    for m in range(idx.shape[0]):
        sel = np.nonzero(np.max(np.abs(centers - idx[m]), axis=1) <= gamma)[0]
        hits[m] = sel.size
        tot = 0.0
        for nu in sel:
            off = idx[m] - centers[nu] + gamma
            tot += z[nu] * float(np.dot(wl, ul[off[0]] * ul[off[1]] * ul[off[2]]))
        out[m] = tot
    return out, hits


# ---------------------------------------------- observables.py:101-259
def self_value(table, w, split_index, h):
    c = table.shape[0] // 2
    u = table[:, :split_index + 1]
    return float(np.dot(w[:split_index + 1], u[c] * u[c] * u[c])) / h ** 3


def rs_energy(core, zs, idx, z, table, w, split_index, h):
    vals = eval_tucker_many(core, zs, idx) / h ** 3
    return 0.5 * math.fsum(z * (vals - z * self_value(table, w, split_index, h)))


def _window_values(table, w, offsets, nt, h):
    c = table.shape[0] // 2
    rows = table[c + offsets[:, 0], :nt] * table[c + offsets[:, 1], :nt] * \
        table[c + offsets[:, 2], :nt]
    return (rows @ w[:nt]) / h ** 3


def reference_energy(idx, z, table, w, split_index, h):
    nt = split_index + 1
    sv = self_value(table, w, split_index, h)
    terms = []
    for j in range(idx.shape[0]):
        p = math.fsum(z * _window_values(table, w, idx[j] - idx, nt, h))
        terms.append(z[j] * (p - z[j] * sv))
    return 0.5 * math.fsum(terms)


def force_fd(idx, z, table, w, split_index, h, j):
    nt = split_index + 1
    others = np.arange(idx.shape[0]) != j
    off = idx[j] - idx[others]
    base = _window_values(table, w, off, nt, h)
    f = np.empty(3)
    for a in range(3):
        sh = off.copy()
        sh[:, a] -= 1
        f[a] = z[j] * math.fsum(z[others] * (_window_values(table, w, sh, nt, h) - base)) / h
    return f


def force_fd_scale(idx, z, table, w, split_index, h, j):
    """Magnitude the differences of force_fd cancel from, per axis:
    |z_j| sum_p |z_p| (|shifted| + |base|) / h (the rounding-error scale of
    observables.py:253-256; used by the tests to state the force tolerance)."""
    nt = split_index + 1
    others = np.arange(idx.shape[0]) != j
    off = idx[j] - idx[others]
    base = np.abs(_window_values(table, w, off, nt, h))
    s = np.empty(3)
    for a in range(3):
        sh = off.copy()
        sh[:, a] -= 1
        s[a] = abs(z[j]) * math.fsum(np.abs(z[others]) * (np.abs(_window_values(table, w, sh, nt, h)) + base)) / h
    return s


# ------------------------------------------------------------ full pipeline
def prologue(kind, lam, b, n, M, split_index, delta, C0=3.0):
    h = grid_h(b, n)
    t, a = quadrature(kind, lam, M, C0, 0.5 * h, 2.0 * math.sqrt(3.0) * b)
    table, w = doubled_table(t, a, b, n)
    gamma = min(max(gamma_of(table, w, split_index, delta, h), 0), n - 1)
    return dict(nodes=t, qweights=a, table=table, w=w, gamma=gamma, h=h)


def build_and_dense(case: dict, ranks=None, dense: bool = True, use_c: bool = True):
    """Reference pipeline with max_sweeps=0 + dense_rs, plain arrays in/out."""
    p = prologue(case["kind"], case.get("lam", 1.0), case["b"], case["n"], case["M"],
                 case["split_index"], case["delta"])
    idx, _, maxd = snap(case["positions"], case["b"], case["n"])
    z = case["charges"]
    weights, facs = long_side_matrices(p["table"], p["w"], idx, z, case["split_index"])
    core, zs, spectra, rk = rhosvd(weights, facs, eps=case.get("eps"), ranks=ranks)
    ul, wl = local_window(p["table"], p["w"], case["split_index"], p["gamma"])
    out = dict(p, idx=idx, core=core, zs=zs, spectra=spectra, ranks=rk, ul=ul, wl=wl,
               max_disp=maxd)
    if dense:
        n = case["n"]
        L0 = local_dense(ul, wl)
        short = dense_cct_c(L0, p["gamma"], idx, z, n) if use_c else \
            dense_cct_numpy(L0, p["gamma"], idx, z, n)
        out["grid"] = tucker_dense(core, zs) + short
    return out


def small_case(n: int = 32, count: int = 24, seed: int = 5, kind: str = "newton"):
    """A tiny random system (uniform cluster, uniform charges) for smoke tests."""
    rng = np.random.default_rng(seed)
    b = 8.0
    h = 2 * b / n
    while True:
        pos = rng.uniform(-0.7 * b, 0.7 * b, (count, 3))
        idx = np.clip(np.ceil(pos / h + n // 2 - 0.5).astype(np.int64), 1, n - 1)
        if np.unique(idx, axis=0).shape[0] == count:
            break
    q = rng.uniform(-1.0, 1.0, count)
    return dict(kind=kind, lam=0.5, b=b, n=n, M=15, split_index=7, delta=1e-6, eps=1e-8,
                positions=pos, charges=q)


# --------------------------------------- large configs: shift-merged RHOSVD
def shift_rhosvd(case: dict, p: dict, idx: np.ndarray, ranks=None, eps=None):
    """RHOSVD of the long part through the exact shift regrouping
    ``A A^T = sum_s c_s sum_k w_k^2 u_k[s:s+n] u_k[s:s+n]^T`` (rankred.py:82-126
    restated; pinned against the literal route at C1/C2 by the tests) -- the
    CPU oracle for C3-C5 where the literal n x N R_l side matrices are 2-44 GB.
    Returns (core, zs, spectra, ranks)."""
    n = case["n"]
    nt = case["split_index"] + 1
    table, w = p["table"], p["w"]
    z = case["charges"]
    starts = n - idx
    zs, spectra = [], []
    for l in range(3):
        c = np.zeros(n + 1)
        np.add.at(c, starts[:, l], z * z)
        s_used = np.nonzero(c)[0]
        X = np.concatenate([table[s:s + n, :nt] * (np.sqrt(c[s]) * np.abs(w[:nt]))
                            for s in s_used], axis=1)
        vals, vecs = np.linalg.eigh(X @ X.T)
        order = np.argsort(vals)[::-1]
        vals = np.clip(vals[order], 0.0, None)
        zz = vecs[:, order]
        lead = np.abs(zz).argmax(axis=0)
        sg = np.sign(zz[lead, np.arange(zz.shape[1])])
        sg[sg == 0] = 1.0
        zs.append(zz * sg)
        spectra.append(np.sqrt(vals))
    if ranks is None:
        ranks = tuple(min(eps_rank(s, eps if eps is not None else case["eps"]), n) for s in spectra)
    zs = [zz[:, :r] for zz, r in zip(zs, ranks)]
    # projections per shift: TT[a, s, k] = sum_i Z[i, a] T[s + i, k]
    from numpy.lib.stride_tricks import sliding_window_view
    tts = []
    for zl in zs:
        tt = np.empty((zl.shape[1], n, nt))
        for k in range(nt):
            H = sliding_window_view(table[:, k], n)[:n]   # H[s, i] = T[s + i, k]
            tt[:, :, k] = zl.T @ H.T
        tts.append(tt)
    # core = sum_p z_p sum_k w_k TT1[:, s1p, k] (x) TT2[:, s2p, k] (x) TT3[:, s3p, k]
    r1, r2, r3 = ranks
    core = np.zeros((r1 * r2, r3))
    chunk = max(1, 4096 // nt)
    for p0 in range(0, idx.shape[0], chunk):
        sl = slice(p0, min(idx.shape[0], p0 + chunk))
        P1 = tts[0][:, starts[sl, 0], :] * (z[sl, None] * w[None, :nt])   # (r1, m, nt)
        P2 = tts[1][:, starts[sl, 1], :]
        P3 = tts[2][:, starts[sl, 2], :]
        kr = (P1[:, None] * P2[None, :]).reshape(r1 * r2, -1)
        core += kr @ P3.reshape(r3, -1).T
    return core.reshape(r1, r2, r3), zs, spectra, tuple(ranks)


def slab_grid(case: dict, planes, ranks=None):
    """Oracle grid planes ``planes`` (list of x1 indices) for any config:
    Tucker part from :func:`shift_rhosvd` evaluated on those planes
    (formats.py:173-176 restricted to V1[planes]) + the C dense_cct loop on the
    same planes (formats.py:432-445).  Returns (planes grid, ranks, gamma)."""
    p = prologue(case["kind"], case.get("lam", 1.0), case["b"], case["n"], case["M"],
                 case["split_index"], case["delta"])
    idx, _, _ = snap(case["positions"], case["b"], case["n"])
    core, zs, _, rk = shift_rhosvd(case, p, idx, ranks=ranks)
    ul, wl = local_window(p["table"], p["w"], case["split_index"], p["gamma"])
    L0 = local_dense(ul, wl)
    out = []
    for x in planes:
        t = np.einsum("abc,a,jb,lc->jl", core, zs[0][x], zs[1], zs[2], optimize=True)
        sh = dense_cct_c(L0, p["gamma"], idx, case["charges"], case["n"], x, x + 1)[0]
        out.append(t + sh)
    return np.stack(out), rk, p["gamma"]
