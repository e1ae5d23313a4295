"""Rank-structured tensor formats with device-resident data, and the grid
assembly / point evaluation entry points of the RS path.

Same public names and semantics as the reference ``formats.py``:

* :class:`CanonicalTensor` (``formats.py:44-118``), :class:`TuckerTensor`
  (``:137-176``), :class:`CCT` (``:179-244``), :class:`RSCanonical` /
  :class:`RSTucker` (``:269-308``);
* ``dense_rs`` / ``dense_cct`` / ``TuckerTensor.dense`` (``:173-176, 423-453``)
  -- here ONE fused device pass (``rs_assemble_planes``): every grid point is
  written exactly once as Tucker value + short-range sum, computed as a
  plane GEMM on FP64 tensor cores;
* ``eval_*`` point evaluation (``:321-420``) -- ``rs_eval_tucker`` /
  ``rs_eval_cct``, including the soft-overlap ``CapacityError`` cap.

Arrays may be numpy (host) or torch CUDA tensors; heavy data produced by
this package (side matrices, Tucker factors, grids) stays on the device and
is only copied to the host when a numpy result is requested
(``dense_rs(..., device=False)``, the reference-compatible default).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import os

import numpy as np

from . import _native as nat
from .errors import CapabilityError, CapacityError, ConfigError, DomainError, SeparationError
from .particles import Grid3

MAX_DENSE_ELEMENTS = 128 ** 3
_ASSEMBLE_WORKSPACE = 3 << 30  # bytes of A-operand scratch per chunk of planes


def _torch():
    import torch

    return torch


def is_device(x) -> bool:
    torch = _torch()
    return isinstance(x, torch.Tensor)


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (float64 unless dtype given)."""
    torch = nat._torch()
    dt = dtype or torch.float64
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
        return t.to(dt).contiguous()
    return torch.from_numpy(np.array(x, copy=True, order="C")).to(device="cuda", dtype=dt)


def to_host(x) -> np.ndarray:
    if is_device(x):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _guard_dense(shape, limit: int) -> None:
    total = int(np.prod([int(s) for s in shape]))
    if total > limit:
        raise CapacityError(
            f"refusing to materialize a dense {tuple(int(s) for s in shape)} tensor "
            f"({total} > {limit} elements); raise the limit explicitly if this is intentional")


def _readonly(a):
    if is_device(a):
        return a.contiguous()
    a = np.ascontiguousarray(a)
    a.setflags(write=False)
    return a


# ================================================================ canonical
@dataclass(frozen=True)
class CanonicalTensor:
    """Weights plus one side matrix per mode (host or device arrays)."""

    weights: object
    factors: tuple

    def __post_init__(self):
        w = self.weights
        if is_device(w):
            w = w.reshape(-1).to(_torch().float64).contiguous()
        else:
            w = _readonly(np.asarray(w, dtype=np.float64).reshape(-1))
        facs = []
        for f in self.factors:
            f = f.to(_torch().float64).contiguous() if is_device(f) else _readonly(
                np.asarray(f, dtype=np.float64))
            facs.append(f)
        facs = tuple(facs)
        if len(facs) != 3:
            raise DomainError("canonical tensor needs exactly three side matrices")
        for f in facs:
            if f.ndim != 2 or f.shape[1] != w.shape[0]:
                raise DomainError(f"side matrix shape {tuple(f.shape)} inconsistent with rank "
                                  f"{w.shape[0]}")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "factors", facs)

    @property
    def rank(self) -> int:
        return int(self.weights.shape[0])

    @property
    def mode_sizes(self) -> tuple:
        return tuple(int(f.shape[0]) for f in self.factors)

    @classmethod
    def empty(cls, mode_sizes) -> "CanonicalTensor":
        return cls(np.zeros(0), tuple(np.zeros((int(n), 0)) for n in mode_sizes))

    def normalize(self) -> "CanonicalTensor":
        """Unit columns, norms folded into the weights (``formats.py:80-91``)."""
        if self.rank == 0:
            return self
        if is_device(self.weights):
            torch = _torch()
            w = self.weights.clone()
            facs = []
            for f in self.factors:
                norms = torch.linalg.vector_norm(f, dim=0)
                w = w * norms
                facs.append(f / torch.where(norms > 0, norms, torch.ones_like(norms)))
            return CanonicalTensor(w, tuple(facs))
        w = self.weights.copy()
        facs = []
        for f in self.factors:
            norms = np.linalg.norm(f, axis=0)
            safe = np.where(norms > 0, norms, 1.0)
            w = w * norms
            facs.append(f / safe)
        return CanonicalTensor(w, tuple(facs))

    def dense(self, limit: int = MAX_DENSE_ELEMENTS, device: bool = False):
        """Dense ``sum_k w_k u1 (x) u2 (x) u3`` via the plane GEMM (no short part)."""
        _guard_dense(self.mode_sizes, limit)
        torch = nat._torch()
        n1, n2, n3 = self.mode_sizes
        if self.rank == 0:
            out = torch.zeros((n1, n2, n3), dtype=torch.float64, device="cuda")
            return out if device else to_host(out)
        w = to_device(self.weights)
        u1, u2, u3 = (to_device(f) for f in self.factors)
        kp = self.rank + (self.rank % 2)
        a = torch.zeros((n1 * n2, kp), dtype=torch.float64, device="cuda")
        a[:, : self.rank] = (u1[:, None, :] * w * u2[None, :, :]).reshape(n1 * n2, self.rank)
        b = torch.zeros((n3, kp), dtype=torch.float64, device="cuda")
        b[:, : self.rank] = u3
        out = torch.empty((n1, n2, n3), dtype=torch.float64, device="cuda")
        nat.check(nat.lib().rs_gemm_nt(a.data_ptr(), kp, b.data_ptr(), kp, out.data_ptr(), n3,
                                       n1 * n2, n3, kp, nat.stream_ptr()), "CanonicalTensor.dense")
        return out if device else to_host(out)


# ==================================================================== Tucker
@dataclass(frozen=True)
class TuckerTensor:
    """Core contracted with orthonormal factors (device arrays)."""

    core: object
    factors: tuple

    def __post_init__(self):
        torch = nat._torch()
        core = to_device(self.core)
        facs = tuple(to_device(f) for f in self.factors)
        if core.ndim != 3 or len(facs) != 3:
            raise DomainError("Tucker tensor needs a 3D core and three factors")
        for axis, f in enumerate(facs):
            if f.ndim != 2 or f.shape[1] != core.shape[axis]:
                raise DomainError(f"factor {axis} shape {tuple(f.shape)} inconsistent with core "
                                  f"{tuple(core.shape)}")
            if f.shape[1] > f.shape[0]:
                raise DomainError("Tucker rank exceeds mode size")
            gram = f.T @ f
            eye = torch.eye(f.shape[1], dtype=torch.float64, device=f.device)
            # np.allclose(eye, I, atol=1e-11): |x - y| <= atol + rtol |y|, rtol = 1e-5
            if not bool(torch.all(torch.abs(gram - eye) <= 1e-11 + 1e-5 * eye)):
                raise DomainError(f"factor {axis} columns are not orthonormal")
        object.__setattr__(self, "core", core)
        object.__setattr__(self, "factors", facs)

    @property
    def ranks(self) -> tuple:
        return tuple(int(r) for r in self.core.shape)

    @property
    def mode_sizes(self) -> tuple:
        return tuple(int(f.shape[0]) for f in self.factors)

    def norm(self) -> float:
        return float(_torch().linalg.vector_norm(self.core))

    def dense(self, limit: int = MAX_DENSE_ELEMENTS, device: bool = False):
        _guard_dense(self.mode_sizes, limit)
        out = assemble_grid(self, None)
        return out if device else to_host(out)


# ======================================================================= CCT
def _buckets_host(centers: np.ndarray, gamma: int) -> dict:
    cell = gamma + 1
    keys = centers // cell
    out: dict = {}
    for nu, key in enumerate(map(tuple, keys.tolist())):
        out.setdefault(key, []).append(nu)
    return {k: np.asarray(v, dtype=np.int64) for k, v in out.items()}


@dataclass(frozen=True)
class CCT:
    """Cumulated canonical tensor: the local short-range tensor on a
    ``(2 gamma + 1)^3`` window replicated at ``centers`` with ``weights``."""

    local: CanonicalTensor
    gamma: int
    centers: object
    weights: object
    mode_sizes: tuple
    overlap_policy: str = "soft"
    max_overlap: Optional[int] = 8
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        gamma = int(self.gamma)
        if is_device(self.centers):
            centers = self.centers.reshape(-1, 3).to(_torch().int64).contiguous()
        else:
            centers = _readonly(np.asarray(self.centers, dtype=np.int64).reshape(-1, 3))
        if is_device(self.weights):
            weights = self.weights.reshape(-1).to(_torch().float64).contiguous()
        else:
            weights = _readonly(np.asarray(self.weights, dtype=np.float64).reshape(-1))
        sizes = tuple(int(s) for s in self.mode_sizes)
        if gamma < 0:
            raise DomainError("gamma must be non-negative")
        if centers.shape[0] != weights.shape[0]:
            raise DomainError("one weight per center required")
        if self.local.rank > 0:
            win = 2 * gamma + 1
            if self.local.mode_sizes != (win, win, win):
                raise DomainError(f"local tensor modes {self.local.mode_sizes} do not match "
                                  f"window size {win}")
        if self.overlap_policy not in ("strict", "soft"):
            raise DomainError(f"unknown overlap policy {self.overlap_policy!r}")
        if centers.shape[0]:
            lo = int(centers.min())
            hi_ok = bool((centers < (_torch().tensor(sizes, device=centers.device)
                                     if is_device(centers) else np.array(sizes))).all())
            if lo < 0 or not hi_ok:
                raise DomainError("CCT centers out of the ambient index range")
        object.__setattr__(self, "gamma", gamma)
        object.__setattr__(self, "centers", centers)
        object.__setattr__(self, "weights", weights)
        object.__setattr__(self, "mode_sizes", sizes)
        if self.overlap_policy == "strict" and self.local.rank > 0:
            _check_disjoint(centers, gamma)

    @property
    def count(self) -> int:
        return int(self.centers.shape[0])

    @property
    def local_rank(self) -> int:
        return self.local.rank

    @property
    def _buckets(self) -> dict:
        """Host cell-bucket index (``formats.py:238-244``), built on demand."""
        b = self._cache.get("buckets")
        if b is None:
            b = _buckets_host(to_host(self.centers), self.gamma)
            self._cache["buckets"] = b
        return b

    def device_layout(self):
        """Device data of the fused assembly, cached per CCT: local factors and
        the copies bucketed by x3 index (stable order; bucket table built on the
        device by ``rs_short_layout``, so nothing synchronises the host)."""
        lay = self._cache.get("dev")
        if lay is not None:
            return lay
        torch = nat._torch()
        if self.local.rank > 0:
            f = self.local.factors
            same = all(np.array_equal(to_host(f[0]), to_host(g)) for g in f[1:])
            if not same:
                raise DomainError("fused assembly expects the three local factors to coincide "
                                  "(true for every CCT built by assemble_short)")
        c = to_device(self.centers, torch.int64)
        z = to_device(self.weights)
        lay = short_layout(c, z, self.mode_sizes[2])
        lay.update(ul=to_device(self.local.factors[0]).contiguous(),
                   wl=to_device(self.local.weights).contiguous())
        self._cache["dev"] = lay
        return lay


    def l0_supported(self) -> bool:
        """The dense-L0 gathers fold L0 in x1 and x2: they need the local
        factors symmetric about the window centre (always true for
        ``assemble_short``'s window of the doubled table)."""
        v = self._cache.get("l0_sym")
        if v is None:
            u = np.asarray(to_host(self.local.factors[0]))
            g = self.gamma
            v = self._cache["l0_sym"] = bool(u.shape[0] == 2 * g + 1 and 2 * g + 4 <= 256
                                             and np.array_equal(u[g:], u[g::-1]))
        return v

    def l0_table(self):
        """Dense local tensor L0 for the low-overlap gather (``formats.py:432``:
        ``local.dense()``), built on the device from the normalised factors and
        cached per CCT, in the x1-folded two-copy pair layout of
        ``csrc/rs_l0.cuh``: ``P[par, |a-g|, b, c + 2 - par] = L0[a, b, c]``
        (zero margins), shape ``(2, g+1, 2g+1, 256)``."""
        t = self._cache.get("l0")
        if t is None:
            torch = nat._torch()
            lay = self.device_layout()
            if not self.l0_supported():
                raise DomainError("the dense-L0 gather needs local factors symmetric about "
                                  "the window centre")
            g = self.gamma
            t = torch.empty((2, g + 1, 2 * g + 1, 256), dtype=torch.float64,
                            device=lay["ul"].device)
            assert t.numel() * 8 == nat.lib().rs_short_l0_bytes(g)
            nat.check(nat.lib().rs_short_l0_table(nat.ptr(lay["ul"]), nat.ptr(lay["wl"]),
                                                  self.local.rank, self.gamma, t.data_ptr(),
                                                  nat.stream_ptr()), "rs_short_l0_table")
            self._cache["l0"] = t
        return t


def trusted_cct(local, gamma: int, centers, weights, mode_sizes, overlap_policy="soft",
                max_overlap=8) -> "CCT":
    """CCT from device arrays produced by this package (snapped, in range,
    charges float64): skips the validation probes, which would synchronise."""
    c = object.__new__(CCT)
    for k, v in dict(local=local, gamma=int(gamma), centers=centers, weights=weights,
                     mode_sizes=tuple(int(m) for m in mode_sizes), overlap_policy=overlap_policy,
                     max_overlap=max_overlap, _cache={}).items():
        object.__setattr__(c, k, v)
    return c


def short_layout(centers, z, n: int, cnt3=None, prep=None) -> dict:
    """Copies in bucket order (x3-major, ascending x2 inside a bucket: the row
    builder's binary search relies on it) plus the device bucket table; no
    host synchronisation.  ``prep``: the output of the build path's node sort
    (``rs_prep``), reused when given."""
    torch = nat._torch()
    count = int(centers.shape[0])
    if prep is None:
        order = torch.argsort((centers[:, 2] * n + centers[:, 1]) * n + centers[:, 0], stable=True)
        cs = centers[order]
        c1, c2, zq = (cs[:, 0].to(torch.int32).contiguous(), cs[:, 1].to(torch.int32).contiguous(),
                      z[order].contiguous())
    else:
        c1, c2, zq = prep["c1"], prep["c2"], prep["zq"]
    if cnt3 is None:
        cnt3 = torch.zeros(n, dtype=torch.int32, device="cuda").index_add_(
            0, centers[:, 2], torch.ones(count, dtype=torch.int32, device="cuda"))
    bstart = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    bc3 = torch.empty(n, dtype=torch.int32, device="cuda")
    nb = torch.empty(1, dtype=torch.int32, device="cuda")
    nat.check(nat.lib().rs_short_layout(cnt3.data_ptr(), n, bstart.data_ptr(), bc3.data_ptr(),
                                        nb.data_ptr(), nat.stream_ptr()), "rs_short_layout")
    return dict(c1=c1, c2=c2, zq=zq, bstart=bstart, bc3=bc3, nb=nb,
                nb_max=max(1, min(n, count)), centers=centers, z=z)


def _check_disjoint(centers, gamma: int) -> None:
    """Strict policy: pairwise Chebyshev distance > 2 gamma (``formats.py:247-266``)."""
    c = to_host(centers)
    if c.shape[0] < 2:
        return
    order = np.lexsort((c[:, 2], c[:, 1], c[:, 0]))
    cs = c[order]
    for i in range(cs.shape[0]):
        j = i + 1
        while j < cs.shape[0] and cs[j, 0] - cs[i, 0] <= 2 * gamma:
            if np.max(np.abs(cs[j] - cs[i])) <= 2 * gamma:
                a, b = sorted((int(order[i]), int(order[j])))
                raise SeparationError(f"strict policy: gamma vicinities of particles {a} and {b} "
                                      f"intersect (gamma={gamma})")
            j += 1


# ======================================================================= RS
@dataclass(frozen=True)
class RSCanonical:
    long: CanonicalTensor
    short: CCT
    grid: Grid3

    def __post_init__(self):
        n = self.grid.n
        if self.long.mode_sizes != (n, n, n):
            raise DomainError("long part mode sizes do not match the grid")
        if self.short.mode_sizes != (n, n, n):
            raise DomainError("short part ambient sizes do not match the grid")
        if self.short.local.rank > 0 and 2 * self.short.gamma + 1 > n:
            raise DomainError("short-range window exceeds the grid")

    @property
    def mode_sizes(self) -> tuple:
        return self.long.mode_sizes


@dataclass(frozen=True)
class RSTucker:
    long: TuckerTensor
    short: CCT
    grid: Grid3

    def __post_init__(self):
        n = self.grid.n
        if self.long.mode_sizes != (n, n, n):
            raise DomainError("long part mode sizes do not match the grid")
        if self.short.mode_sizes != (n, n, n):
            raise DomainError("short part ambient sizes do not match the grid")

    @property
    def mode_sizes(self) -> tuple:
        return self.long.mode_sizes


# ============================================================ grid assembly
_ASM_PLANS: dict = {}   # (sizes, flags) -> (planes per chunk, workspace bytes)


def assemble_grid(long: Optional[TuckerTensor], short: Optional[CCT], x1_lo: int = 0,
                  x1_hi: Optional[int] = None, out=None, accumulate: bool = False,
                  workspace_bytes: int = _ASSEMBLE_WORKSPACE, workspace_slot: str = "assemble"):
    """x1-planes ``[x1_lo, x1_hi)`` of Tucker(long) + dense(short) on the device
    (either part may be None; ``accumulate`` adds into ``out``).

    One ``rs_assemble_planes`` launch sequence per chunk of planes; every grid
    point is written once, in C order, by the plane GEMM's epilogue.
    """
    torch = nat._torch()
    if long is not None:
        n = long.mode_sizes[0]
        if long.mode_sizes != (n, n, n):
            raise CapabilityError("fused assembly expects a cubic grid")
    elif short is not None:
        n = short.mode_sizes[0]
    else:
        raise DomainError("assemble_grid needs a long or a short part")
    x1_hi = n if x1_hi is None else int(x1_hi)
    if not (0 <= x1_lo < x1_hi <= n):
        raise DomainError(f"bad plane range [{x1_lo}, {x1_hi})")
    planes = x1_hi - x1_lo
    if out is None:
        out = (torch.zeros if accumulate else torch.empty)((planes, n, n), dtype=torch.float64,
                                                           device="cuda")
    flags = nat.ASM_ACCUMULATE if accumulate else 0
    if long is not None:
        flags |= nat.ASM_LONG
        r1, r2, r3 = long.ranks
        core, (v1, v2, v3) = long.core, long.factors
    else:
        r1 = r2 = r3 = 1
        core = v1 = v2 = v3 = None
    have_short = short is not None and short.local.rank > 0 and short.count > 0
    L = nat.lib()
    if have_short and L.rs_short_method(n, short.count, short.gamma,
                                        short.local.rank) == nat.SHORT_L0 \
            and short.l0_supported() and n % 2 == 0:
        # low window overlap: the short part is a dense-L0 gather.  With a long
        # part and no accumulation, both go through ONE pass that stores every
        # grid value once (rs_assemble_fused_l0); otherwise the Tucker planes by
        # the plane GEMM, then the gather on top (rs_assemble_short_l0)
        if (long is not None and not accumulate and _FUSED_L0
                and L.rs_fused_l0_supported(n, long.ranks[2], short.gamma)):
            return _assemble_fused_l0(long, short, x1_lo, x1_hi, out, workspace_bytes,
                                      workspace_slot)
        if long is not None:
            assemble_grid(long, None, x1_lo, x1_hi, out=out, accumulate=accumulate,
                          workspace_bytes=workspace_bytes, workspace_slot=workspace_slot)
        lay = short.device_layout()
        l0 = short.l0_table()
        stream = nat.stream_ptr()
        nat.check(L.rs_assemble_short_l0(
            nat.ptr(l0), short.gamma, n, nat.ptr(lay["c1"]), nat.ptr(lay["c2"]),
            nat.ptr(lay["zq"]), nat.ptr(lay["bstart"]), nat.ptr(lay["bc3"]), nat.ptr(lay["nb"]),
            x1_lo, x1_hi, 1 if (accumulate or long is not None) else 0, out.data_ptr(), stream),
            "rs_assemble_short_l0")
        return out
    if have_short and L.rs_short_method(n, short.count, short.gamma,
                                        short.local.rank) == nat.SHORT_MMA:
        # the fused tensor-core kernel (rs_assemble_short_mma); the Tucker planes,
        # if any, first, then the short part on top
        if long is not None:
            assemble_grid(long, None, x1_lo, x1_hi, out=out, accumulate=accumulate,
                          workspace_bytes=workspace_bytes, workspace_slot=workspace_slot)
        lay = short.device_layout()
        ws = nat.Workspace.get(L.rs_short_mma_workspace_bytes(n, short.gamma), "short_mma")
        nat.check(L.rs_assemble_short_mma(
            nat.ptr(lay["ul"]), nat.ptr(lay["wl"]), short.local.rank, short.gamma, n, short.count,
            nat.ptr(lay["c1"]), nat.ptr(lay["c2"]), nat.ptr(lay["zq"]), nat.ptr(lay["bstart"]),
            nat.ptr(lay["bc3"]), nat.ptr(lay["nb"]), x1_lo, x1_hi,
            nat.ASM_ACCUMULATE if (accumulate or long is not None) else 0, out.data_ptr(),
            ws.data_ptr(), ws.numel(), nat.stream_ptr()), "rs_assemble_short_mma")
        return out
    if have_short:
        flags |= nat.ASM_SHORT | nat.asm_oz(nat.OZ_SLICES)
        lay = short.device_layout()
        rs, gamma, nb_max = short.local.rank, short.gamma, lay["nb_max"]
        ul, wl = lay["ul"], lay["wl"]
        c1, c2, zq, bstart, bc3, nb = (lay[k] for k in ("c1", "c2", "zq", "bstart", "bc3", "nb"))
    else:
        rs, gamma, nb_max = 0, 0, 0
        ul = wl = c1 = c2 = zq = bstart = bc3 = nb = None
    if not (flags & (nat.ASM_LONG | nat.ASM_SHORT)):
        if not accumulate:
            out.zero_()
        return out
    rmax = max(r1, r2, r3)
    key = (n, planes, rmax, nb_max, rs, flags, workspace_bytes)
    plan = _ASM_PLANS.get(key)
    if plan is None:
        one = L.rs_assemble_workspace_bytes(n, 1, rmax, nb_max, rs, flags)
        per_plane = L.rs_assemble_workspace_bytes(n, 2, rmax, nb_max, rs, flags) - one
        fixed = one - per_plane
        chunk = max(1, min(planes, (workspace_bytes - fixed) // max(per_plane, 1)))
        plan = _ASM_PLANS[key] = (chunk, L.rs_assemble_workspace_bytes(n, chunk, rmax, nb_max,
                                                                        rs, flags))
    chunk = plan[0]
    ws = nat.Workspace.get(plan[1], workspace_slot)
    stream = nat.stream_ptr()
    for p0 in range(x1_lo, x1_hi, chunk):
        p1 = min(x1_hi, p0 + chunk)
        dst = out[p0 - x1_lo]
        nat.check(L.rs_assemble_planes(
            nat.ptr(core), r1, r2, r3, nat.ptr(v1), nat.ptr(v2), nat.ptr(v3), n, nat.ptr(ul),
            nat.ptr(wl), rs, gamma, nat.ptr(c1), nat.ptr(c2), nat.ptr(zq), nat.ptr(bstart),
            nat.ptr(bc3), nat.ptr(nb), nb_max, p0, p1, flags, dst.data_ptr(), ws.data_ptr(),
            ws.numel(), stream), "rs_assemble_planes")
    return out


_FUSED_L0 = os.environ.get("RSB200_FUSED", "1") == "1"


def _assemble_fused_l0(long: TuckerTensor, short: CCT, x1_lo: int, x1_hi: int, out,
                       workspace_bytes: int, workspace_slot: str):
    """Tucker + dense-L0 short part in one pass per chunk of planes: the
    per-plane Tucker operands (``RS_ASM_F_ONLY``), then ``rs_assemble_fused_l0``."""
    n = long.mode_sizes[0]
    r1, r2, r3 = long.ranks
    L = nat.lib()
    chunk, wsb = tucker_plan(n, x1_hi - x1_lo, max(r1, r2, r3), workspace_bytes)
    ws = nat.Workspace.get(wsb, workspace_slot)
    core, (v1, v2, v3) = long.core, long.factors
    lay = short.device_layout()
    l0 = short.l0_table()
    stream = nat.stream_ptr()
    for p0 in range(x1_lo, x1_hi, chunk):
        p1 = min(x1_hi, p0 + chunk)
        nat.check(L.rs_assemble_planes(
            core.data_ptr(), r1, r2, r3, v1.data_ptr(), v2.data_ptr(), v3.data_ptr(), n, None,
            None, 0, 0, None, None, None, None, None, None, 0, p0, p1,
            nat.ASM_LONG | nat.ASM_ACCUMULATE | nat.ASM_F_ONLY, out[p0 - x1_lo].data_ptr(),
            ws.data_ptr(), ws.numel(), stream), "rs_assemble_planes")
        nat.check(L.rs_assemble_fused_l0(
            r1, r2, r3, v3.data_ptr(), n, nat.ptr(l0), short.gamma, nat.ptr(lay["c1"]),
            nat.ptr(lay["c2"]), nat.ptr(lay["zq"]), nat.ptr(lay["bstart"]), nat.ptr(lay["bc3"]),
            nat.ptr(lay["nb"]), p0, p1, p0, p1, out[p0 - x1_lo].data_ptr(), ws.data_ptr(),
            ws.numel(), stream), "rs_assemble_fused_l0")
    return out


def tucker_plan(n: int, planes: int, rmax: int, workspace_bytes: int = _ASSEMBLE_WORKSPACE,
                flags: Optional[int] = None):
    """(planes per chunk, workspace bytes) of a Tucker-only accumulate."""
    if flags is None:
        flags = nat.ASM_LONG | nat.ASM_ACCUMULATE
    key = (n, planes, rmax, 0, 0, flags, workspace_bytes)
    plan = _ASM_PLANS.get(key)
    if plan is None:
        L = nat.lib()
        one = L.rs_assemble_workspace_bytes(n, 1, rmax, 0, 0, flags)
        per_plane = L.rs_assemble_workspace_bytes(n, 2, rmax, 0, 0, flags) - one
        chunk = max(1, min(planes, (workspace_bytes - (one - per_plane)) // max(per_plane, 1)))
        plan = _ASM_PLANS[key] = (chunk, L.rs_assemble_workspace_bytes(n, chunk, rmax, 0, 0,
                                                                        flags))
    return plan


def tucker_accumulate(long: TuckerTensor, x1_lo: int, x1_hi: int, out,
                      workspace_bytes: int = _ASSEMBLE_WORKSPACE, workspace_slot: str = "assemble"):
    """``out[x1 - x1_lo] += Tucker(long)[x1]`` for x1 in [x1_lo, x1_hi): the
    long-only case of :func:`assemble_grid` with the argument marshalling cut
    to one cached plan (it runs on build_rs's critical path)."""
    n = long.mode_sizes[0]
    r1, r2, r3 = long.ranks
    planes = x1_hi - x1_lo
    flags = nat.ASM_LONG | nat.ASM_ACCUMULATE
    L = nat.lib()
    chunk, wsb = tucker_plan(n, planes, max(r1, r2, r3), workspace_bytes, flags)
    ws = nat.Workspace.get(wsb, workspace_slot)
    core, (v1, v2, v3) = long.core, long.factors
    cp, p1_, p2_, p3_ = core.data_ptr(), v1.data_ptr(), v2.data_ptr(), v3.data_ptr()
    wp, wn, st = ws.data_ptr(), ws.numel(), nat.stream_ptr()
    base, pstride = out.data_ptr(), n * n * 8
    for p0 in range(x1_lo, x1_hi, chunk):
        p1 = min(x1_hi, p0 + chunk)
        nat.check(L.rs_assemble_planes(cp, r1, r2, r3, p1_, p2_, p3_, n, None, None, 0, 0, None,
                                       None, None, None, None, None, 0, p0, p1, flags,
                                       base + (p0 - x1_lo) * pstride, wp, wn, st),
                  "rs_assemble_planes")
    return out


def dense_cct(short: CCT, limit: int = MAX_DENSE_ELEMENTS, device: bool = False):
    """Dense short-range sum (``formats.py:432-445``): windows clipped at the faces."""
    _guard_dense(short.mode_sizes, limit)
    torch = nat._torch()
    n = short.mode_sizes[0]
    if short.local.rank == 0:
        out = torch.zeros(short.mode_sizes, dtype=torch.float64, device="cuda")
        return out if device else to_host(out)
    _guard_dense(short.local.mode_sizes, limit)
    out = assemble_grid(None, short)
    return out if device else to_host(out)


_PINNED: dict = {}          # shape -> pinned host tensor we may hand out again
_HOST_CHUNKS = 8            # plane chunks of the overlapped device->host path


def _pinned_host(shape):
    """A pinned host float64 tensor of ``shape``; the previous one is reused
    once every numpy view handed out from it is gone (weak liveness token)."""
    torch = nat._torch()
    ent = _PINNED.get(shape)
    if ent is not None and (ent[1] is None or ent[1]() is None):
        return ent[0]
    t = torch.empty(shape, dtype=torch.float64, pin_memory=True)
    _PINNED[shape] = (t, None)
    return t


def _hand_out(t) -> np.ndarray:
    """numpy view of a pooled pinned tensor; its base (a tensor wrapper kept
    alive by every derived view) becomes the buffer's liveness token."""
    import weakref
    arr = t.numpy()
    key = tuple(t.shape)
    if key in _PINNED and _PINNED[key][0] is t:
        _PINNED[key] = (t, weakref.ref(arr.base))
    return arr


def _copy_stream():
    torch = nat._torch()
    dev = torch.cuda.current_device()
    st = _PINNED.get(("copy", dev))
    if st is None:
        st = torch.cuda.Stream(device=dev)
        _PINNED[("copy", dev)] = st
    return st


def _dense_to_host(a: "RSTucker", lo: int, hi: int, out=None):
    """Planes ``[lo, hi)`` into pinned host memory, chunk by chunk: the
    device->host copy of chunk k (on a copy stream) overlaps the assembly of
    chunk k+1, so the transfer -- the bound of a host-returning call -- starts
    as soon as the first planes exist.  Two rotating device chunk buffers."""
    torch = nat._torch()
    n = a.grid.n
    planes = hi - lo
    host = out if out is not None else _pinned_host((planes, n, n))
    chunk = max(1, -(-planes // _HOST_CHUNKS))
    main = torch.cuda.current_stream()
    cp = _copy_stream()
    bufs = [torch.empty((chunk, n, n), dtype=torch.float64, device="cuda") for _ in range(2)]
    free = [None, None]            # copy-done events guarding buffer reuse
    for i, p0 in enumerate(range(lo, hi, chunk)):
        p1 = min(hi, p0 + chunk)
        b = bufs[i % 2]
        if free[i % 2] is not None:
            main.wait_event(free[i % 2])
        assemble_grid(a.long, a.short, p0, p1, out=b[: p1 - p0])
        ready = torch.cuda.Event()
        ready.record(main)
        cp.wait_event(ready)
        with torch.cuda.stream(cp):
            host[p0 - lo:p1 - lo].copy_(b[: p1 - p0], non_blocking=True)
            done = torch.cuda.Event()
            done.record(cp)
        free[i % 2] = done
        b.record_stream(cp)
    cp.synchronize()
    return host


def dense_rs(a, limit: int = MAX_DENSE_ELEMENTS, device: bool = False, x1_range=None, out=None):
    """Dense RS tensor ``long + short`` (``formats.py:448-453``), fused on device.

    ``device=True`` returns the CUDA tensor (grids larger than host RAM);
    the default returns a numpy array like the reference, streamed to pinned
    host memory chunk by chunk while later chunks are still being assembled
    (``out``: an optional pinned host tensor of the result shape to fill).
    ``x1_range`` (extension) assembles only the x1 planes ``[lo, hi)``
    (multi-GPU slabs).  If :func:`build_rs` prefetched the short-range
    planes, only the Tucker part is added here.
    """
    if isinstance(a, RSTucker):
        _guard_dense(a.long.mode_sizes, limit)
        if a.short.local.rank > 0:
            _guard_dense(a.short.local.mode_sizes, limit)
        n = a.grid.n
        lo, hi = (0, n) if x1_range is None else (int(x1_range[0]), int(x1_range[1]))
        pre = a.short._cache.get("prefetch")
        if pre is not None and pre["lo"] == lo and pre["hi"] == hi:
            del a.short._cache["prefetch"]
            torch = nat._torch()
            res = pre["buf"]
            if not device and pre["complete"] and pre["groups"] is not None:
                # finished group by group (build_rs): each group's D2H starts
                # as soon as its planes are final
                host = out if out is not None else _pinned_host((hi - lo, n, n))
                cp = _copy_stream()
                grp, done = pre["groups"]
                for g, ev in enumerate(done):
                    g0, g1 = g * grp, min(hi - lo, (g + 1) * grp)
                    cp.wait_event(ev)
                    with torch.cuda.stream(cp):
                        host[g0:g1].copy_(res[g0:g1], non_blocking=True)
                res.record_stream(cp)
                cp.synchronize()
                arr = _hand_out(host)
                return arr.reshape(n, n, n) if x1_range is None else arr
            main = torch.cuda.current_stream()
            main.wait_event(pre["ev"])
            res.record_stream(main)
            if not pre["complete"]:  # short part only so far: add the Tucker part
                assemble_grid(a.long, None, lo, hi, out=res, accumulate=True)
        elif not device:
            host = _dense_to_host(a, lo, hi, out)
            arr = _hand_out(host)
            return arr.reshape(n, n, n) if x1_range is None else arr
        else:
            res = assemble_grid(a.long, a.short, lo, hi)
        if x1_range is None:
            res = res.view(n, n, n)
        if device:
            return res
        if out is not None:
            out.copy_(res.reshape(out.shape))
            return out.numpy()
        return to_host(res)
    if isinstance(a, RSCanonical):
        long = a.long.dense(limit=limit, device=True)
        short = dense_cct(a.short, limit=limit, device=True)
        res = long.add_(short)
        return res if device else to_host(res)
    raise ConfigError(f"dense_rs expects an RS tensor, got {type(a).__name__}")


# ======================================================= point evaluation
def _check_index(i, mode_sizes) -> tuple:
    i = tuple(int(v) for v in i)
    if len(i) != 3:
        raise DomainError(f"expected a 3D multi-index, got {i}")
    for v, n in zip(i, mode_sizes):
        if v < 0 or v >= n:
            raise IndexError(f"index {i} out of range for modes {mode_sizes}")
    return i


def _index_tensor(idx, mode_sizes):
    torch = nat._torch()
    t = to_device(idx, torch.int64).reshape(-1, 3)
    if t.shape[0]:
        sizes = torch.tensor(mode_sizes, device="cuda")
        bad = ((t < 0) | (t >= sizes)).any(dim=1)
        if bool(bad.any()):
            k = int(torch.nonzero(bad)[0, 0])
            raise IndexError(f"index {tuple(to_host(t[k]).tolist())} out of range for modes "
                             f"{mode_sizes}")
    return t.contiguous()


def eval_tucker_many(t: TuckerTensor, idx, device: bool = False):
    torch = nat._torch()
    it = _index_tensor(idx, t.mode_sizes)
    out = torch.empty(it.shape[0], dtype=torch.float64, device="cuda")
    r1, r2, r3 = t.ranks
    v1, v2, v3 = t.factors
    nat.check(nat.lib().rs_eval_tucker(t.core.data_ptr(), r1, r2, r3, v1.data_ptr(), v2.data_ptr(),
                                       v3.data_ptr(), it.data_ptr(), it.shape[0], out.data_ptr(),
                                       nat.stream_ptr()), "rs_eval_tucker")
    return out if device else to_host(out)


def eval_tucker(t: TuckerTensor, i) -> float:
    i = _check_index(i, t.mode_sizes)
    return float(eval_tucker_many(t, np.asarray([i]))[0])


def eval_canonical_many(t: CanonicalTensor, idx, device: bool = False):
    torch = nat._torch()
    it = _index_tensor(idx, t.mode_sizes)
    if t.rank == 0:
        out = torch.zeros(it.shape[0], dtype=torch.float64, device="cuda")
    else:
        u = [to_device(f) for f in t.factors]
        rows = u[0][it[:, 0]] * u[1][it[:, 1]] * u[2][it[:, 2]]
        out = rows @ to_device(t.weights)
    return out if device else to_host(out)


def eval_canonical(t: CanonicalTensor, i) -> float:
    i = _check_index(i, t.mode_sizes)
    return float(eval_canonical_many(t, np.asarray([i]))[0])


def _cct_values(short: CCT, it):
    """(values, hits) of the short part at device indices ``it``."""
    torch = nat._torch()
    m = it.shape[0]
    vals = torch.zeros(m, dtype=torch.float64, device="cuda")
    hits = torch.zeros(m, dtype=torch.int32, device="cuda")
    if short.local.rank == 0 or short.count == 0 or m == 0:
        return vals, hits
    lay = short.device_layout()
    nat.check(nat.lib().rs_eval_cct(lay["ul"].data_ptr(), lay["wl"].data_ptr(), short.local.rank,
                                    short.gamma, lay["centers"].data_ptr(), lay["z"].data_ptr(),
                                    short.count, it.data_ptr(), m, vals.data_ptr(),
                                    hits.data_ptr(), nat.stream_ptr()), "rs_eval_cct")
    return vals, hits


def _apply_overlap_cap(short: CCT, it, hits) -> None:
    if short.max_overlap is None or short.local.rank == 0:
        return
    torch = nat._torch()
    over = hits > short.max_overlap
    if bool(over.any()):
        k = int(torch.nonzero(over)[0, 0])
        i = tuple(to_host(it[k]).tolist())
        raise CapacityError(f"{int(hits[k])} overlapping short-range copies at {i} exceed the "
                            f"soft-policy cap {short.max_overlap}")


def lookup_short(short: CCT, i) -> np.ndarray:
    """Copies whose gamma vicinity contains ``i``, ascending (``formats.py:355-377``)."""
    i = np.asarray(i, dtype=np.int64).reshape(3)
    if short.count == 0:
        return np.zeros(0, dtype=np.int64)
    c = to_host(short.centers)
    sel = np.max(np.abs(c - i), axis=1) <= short.gamma
    return np.flatnonzero(sel).astype(np.int64)


def eval_cct(short: CCT, i) -> float:
    i = _check_index(i, short.mode_sizes)
    if short.local.rank == 0:
        return 0.0
    it = to_device(np.asarray([i]), nat._torch().int64)
    vals, hits = _cct_values(short, it)
    _apply_overlap_cap(short, it, hits)
    return float(vals[0])


def eval_rs(a, i) -> float:
    if isinstance(a, RSCanonical):
        return eval_canonical(a.long, i) + eval_cct(a.short, i)
    if isinstance(a, RSTucker):
        return eval_tucker(a.long, i) + eval_cct(a.short, i)
    raise ConfigError(f"eval_rs expects an RS tensor, got {type(a).__name__}")


def eval_rs_many(a, idx, device: bool = False):
    """RS values at an (m, 3) index array (``formats.py:410-420``)."""
    if isinstance(a, RSCanonical):
        longv = eval_canonical_many(a.long, idx, device=True)
    elif isinstance(a, RSTucker):
        longv = eval_tucker_many(a.long, idx, device=True)
    else:
        raise ConfigError(f"eval_rs_many expects an RS tensor, got {type(a).__name__}")
    if a.short.local.rank > 0:
        it = _index_tensor(idx, a.mode_sizes)
        sv, hits = _cct_values(a.short, it)
        _apply_overlap_cap(a.short, it, hits)
        longv = longv + sv
    return longv if device else to_host(longv)


# ================================================================ storage
@dataclass(frozen=True)
class StorageReport:
    long_floats: int
    short_floats: int
    particle_floats: int
    normal_form_extra: int
    bound: int

    @property
    def total(self) -> int:
        return self.long_floats + self.short_floats + self.particle_floats

    @property
    def within_bound(self) -> bool:
        return self.total <= self.bound


def storage_report(a) -> StorageReport:
    """Float count of an RS tensor (``formats.py:597-625``, same convention)."""
    d = 3
    short = a.short
    window = 2 * short.gamma + 1 if short.local.rank > 0 else 0
    short_floats = d * short.local.rank * window
    particle_floats = (d + 1) * short.count
    if isinstance(a, RSCanonical):
        n = a.long.mode_sizes[0]
        long_floats = d * a.long.rank * n
        extra = a.long.rank + short.local.rank
        bound = d * a.long.rank * n + (d + 1) * short.count + d * short.local.rank * window
    elif isinstance(a, RSTucker):
        r1, r2, r3 = a.long.ranks
        long_floats = r1 * r2 * r3 + sum(r * m for r, m in zip(a.long.ranks, a.long.mode_sizes))
        extra = short.local.rank
        bound = long_floats + (d + 1) * short.count + d * short.local.rank * window
    else:
        raise ConfigError(f"storage_report expects an RS tensor, got {type(a).__name__}")
    return StorageReport(long_floats=long_floats, short_floats=short_floats,
                         particle_floats=particle_floats, normal_form_extra=extra, bound=bound)
