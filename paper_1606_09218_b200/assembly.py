"""RS tensor construction: the reference's ``build_rs`` pipeline on the device.

Reference: ``assembly.py:39-279``.  Per grid configuration the host prologue
(quadrature, ``(2n, R)`` table, split, gamma, normalised short window) is
computed once and cached in an :class:`RSPlan` (it never depends on the
particles).  Per particle system everything runs on the device:

1. snap (``rs_snap``) and the duplicate-node check,
2. per-mode shift histograms and the shift-merged Gram (``rs_gather_windows``
   + ``rs_syrk`` on DMMA), cuSOLVER ``eigh``,
3. ONE host synchronisation: spectra (for the eps-rank rule), collision flag,
   max displacement,
4. shift projection + RHOSVD core (``rs_shift_project`` + ``rs_core``),
5. the CCT short part (centres/charges stay on the device).

The long side matrices of ``assemble_long`` are never materialised on this
path; ``assemble_long`` itself (public API) materialises them on the device
with ``rs_gather_windows`` for callers that want them.
"""

from __future__ import annotations

import os

import dataclasses
import math
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _native as nat
from .errors import ConfigError, DomainError, ResolutionError
from .formats import tucker_accumulate, tucker_plan, CCT, CanonicalTensor, RSCanonical, RSTucker, assemble_grid, is_device, \
    short_layout, storage_report, to_device, to_host, trusted_cct
from .parallel import particle_shard, sharded_sum
from .particles import Grid3, IndexedParticleSystem, ParticleSystem, separation_distance, \
    snap_to_grid
from .quadrature import RadialKernel, ReferenceCanonical, build_quadrature, effective_support, \
    project_kernel, split_rank, split_tensor
from .rankred import TOPEIG_BLOCK, TOPEIG_ITERS, TOPEIG_MAX_BLOCK, TOPEIG_WIDE_BLOCK, ReductionConfig, top_eig_supported, \
    SvdSpectrum, _trusted_tucker, c2t_als, eig_desc, eig_desc_batched, eps_rank, rhosvd_error_bound, shift_histograms, \
    shifted_core, shifted_grams, side_svd, top_eig, rank_rule_fast, truncated_spectrum, tucker_to_canonical


@dataclass(frozen=True)
class AssemblyConfig:
    """Pipeline configuration, same fields/defaults as ``assembly.py:39-69``."""

    grid: Grid3
    kernel: RadialKernel = field(default_factory=lambda: RadialKernel("newton"))
    M: int = 25
    C0: float = 3.0
    split_index: Optional[int] = None
    sigma: Optional[float] = None
    delta: float = 1e-4
    criterion: str = "max_norm"
    overlap_policy: str = "soft"
    max_overlap: Optional[int] = 8
    reduction: ReductionConfig = field(default_factory=lambda: ReductionConfig(eps=1e-5))
    long_format: str = "canonical"
    entry_rule: str = "integral"
    reduce_long: Optional[bool] = None
    reduce_threshold: int = 2000

    def __post_init__(self):
        if self.long_format not in ("canonical", "tucker"):
            raise ConfigError(f"unknown long format {self.long_format!r}")
        if not (0 < self.delta < 1):
            raise ConfigError(f"delta must lie in (0,1), got {self.delta}")


def reference_for(cfg: AssemblyConfig) -> ReferenceCanonical:
    """Doubled-grid reference calibrated on ``[h/2, 2 sqrt(3) b]`` (``assembly.py:72-82``)."""
    b = cfg.grid.box.half_width
    rule = build_quadrature(cfg.kernel, cfg.M, cfg.C0,
                            r_range=(0.5 * cfg.grid.h, 2.0 * math.sqrt(3.0) * b))
    return project_kernel(rule, cfg.grid, doubled=True, entry_rule=cfg.entry_rule)


def window_slice(ref2n: ReferenceCanonical, j, k: int):
    """Mode vectors of one windowed term: slices of the table (``assembly.py:85-98``)."""
    if not ref2n.doubled:
        raise ConfigError("windowing requires the doubled-grid reference")
    n = ref2n.grid.n // 2
    j = tuple(int(v) for v in j)
    if len(j) != 3 or any(v < 0 or v >= n for v in j):
        raise DomainError(f"particle index {j} outside the n-grid")
    return tuple(ref2n.tensor.factors[l][n - j[l]:2 * n - j[l], k] for l in range(3))


# ----------------------------------------------------------------- the plan
@dataclass
class RSPlan:
    """Per-configuration device state: everything ``build_rs`` needs that does
    not depend on the particle set.  Cached by :func:`plan_for`."""

    ref2n: ReferenceCanonical
    split_index: int
    gamma: int
    local: CanonicalTensor          # normalised short window (host)
    table_dev: object               # (2n, R) float64 CUDA
    w_long: object                  # (R_l,) weights
    w_long_abs: object
    local_ul: object = None         # (W, R_s) device copy of the local factor
    local_wl: object = None

    @property
    def n(self) -> int:
        return self.ref2n.grid.n // 2


_QUAD_CACHE: dict = {}
_PLAN_CACHE: dict = {}


def _reference_cached(cfg: AssemblyConfig) -> ReferenceCanonical:
    key = (cfg.grid, cfg.kernel, cfg.M, cfg.C0, cfg.entry_rule)
    ref = _QUAD_CACHE.get(key)
    if ref is None:
        ref = reference_for(cfg)
        _QUAD_CACHE[key] = ref
    return ref


def _short_window(ref2n: ReferenceCanonical, split_index: int, delta: float, gamma=None):
    """(gamma, normalised local tensor) exactly as ``assembly.py:139-184``."""
    n = ref2n.grid.n // 2
    short, _ = split_tensor(ref2n, split_index)
    if short.rank == 0:
        return 0, CanonicalTensor.empty((1, 1, 1))
    if gamma is None:
        gamma = effective_support(short, delta, ref2n.grid.h)
    gamma = int(min(max(gamma, 0), n - 1))
    n0 = ref2n.origin_index
    local = CanonicalTensor(short.weights, tuple(f[n0 - gamma:n0 + gamma + 1, :]
                                                 for f in short.factors)).normalize()
    return gamma, local


def plan_for(cfg: AssemblyConfig, split_index: int) -> RSPlan:
    key = (cfg.grid, cfg.kernel, cfg.M, cfg.C0, cfg.entry_rule, int(split_index), cfg.delta)
    plan = _PLAN_CACHE.get(key)
    if plan is not None:
        return plan
    ref = dataclasses.replace(_reference_cached(cfg), split_index=int(split_index))
    gamma, local = _short_window(ref, split_index, cfg.delta)
    torch = nat._torch()
    table = to_device(ref.table)
    w = to_device(ref.tensor.weights[: split_index + 1])
    plan = RSPlan(ref2n=ref, split_index=int(split_index), gamma=gamma, local=local,
                  table_dev=table, w_long=w, w_long_abs=w.abs().contiguous(),
                  local_ul=to_device(local.factors[0]), local_wl=to_device(local.weights))
    _PLAN_CACHE[key] = plan
    return plan


# ---------------------------------------------------------- particle input
@dataclass(frozen=True)
class DeviceParticles:
    """Device-resident particle system (positions ``(N,3)``, charges ``(N,)``,
    CUDA float64) -- the zero-copy input of :func:`build_rs`."""

    positions: object
    charges: object
    box: object

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


@dataclass(frozen=True)
class DeviceIndexedSystem:
    """Snapped device particle system; host views are materialised lazily."""

    positions: object     # snapped positions (device)
    charges: object       # (device)
    grid: Grid3
    indices: object       # (N, 3) int64 (device)
    box: object
    _disp: object = None  # (N,) displacement (device)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def count(self) -> int:
        return int(self.indices.shape[0])

    @property
    def max_displacement(self) -> float:
        v = self._cache.get("maxdisp")
        if v is None:
            v = float(self._disp.max())
            self._cache["maxdisp"] = v
        return v

    @property
    def base(self) -> ParticleSystem:
        b = self._cache.get("base")
        if b is None:
            b = ParticleSystem(to_host(self.positions), to_host(self.charges), self.box)
            self._cache["base"] = b
        return b

    def to_indexed(self) -> IndexedParticleSystem:
        return IndexedParticleSystem(base=self.base, grid=self.grid, indices=to_host(self.indices),
                                     max_displacement=self.max_displacement)


def snap_device(positions, charges, box, grid: Grid3) -> DeviceIndexedSystem:
    """``rs_snap`` on device data; the collision check is deferred to the
    caller's next synchronisation (see :func:`_collision_flag`)."""
    torch = nat._torch()
    pos = to_device(positions)
    z = to_device(charges)
    count = int(pos.shape[0])
    idx = torch.empty((count, 3), dtype=torch.int64, device="cuda")
    disp = torch.empty(count, dtype=torch.float64, device="cuda")
    key = torch.empty(count, dtype=torch.int64, device="cuda")
    snapped = torch.empty((count, 3), dtype=torch.float64, device="cuda")
    _mark("snap_alloc")
    nat.check(nat.lib().rs_snap(pos.data_ptr(), count, grid.h, grid.n, idx.data_ptr(),
                                disp.data_ptr(), key.data_ptr(), snapped.data_ptr(),
                                nat.stream_ptr()), "rs_snap")
    ds = DeviceIndexedSystem(positions=snapped, charges=z, grid=grid, indices=idx, box=box,
                             _disp=disp)
    ds._cache["key"] = key
    _mark("snap_done")
    return ds


def _node_sort(ds, n: int):
    """One device sort of the particles by node key ``(x3, x2, x1)`` (x3-major)
    plus ``rs_prep``: the bucket-ordered copies (the x3 buckets of the
    short-range layout, ascending x2 inside a bucket as the row builder's
    binary search needs), window starts, the first duplicated node key (-1 if
    none) and the max snap displacement -- all on the device, no sync."""
    torch = nat._torch()
    idx, z = ds.indices, ds.charges
    key = ds._cache.get("key")
    if key is None:
        key = (idx[:, 2] * n + idx[:, 1]) * n + idx[:, 0]
    count = int(idx.shape[0])
    _mark("sort_in")
    ks, order = torch.sort(key, stable=True)
    _mark("sorted")
    c1s = torch.empty(count, dtype=torch.int32, device="cuda")
    c2s = torch.empty(count, dtype=torch.int32, device="cuda")
    zqs = torch.empty(count, dtype=torch.float64, device="cuda")
    starts = torch.empty((count, 3), dtype=torch.int64, device="cuda")
    scal = torch.empty(2, dtype=torch.int64, device="cuda")
    disp = ds._disp if ds._disp is not None and ds._disp.numel() == count else \
        torch.zeros(count, dtype=torch.float64, device="cuda")
    nat.check(nat.lib().rs_prep(ks.data_ptr(), order.data_ptr(), idx.data_ptr(), z.data_ptr(),
                                disp.data_ptr(), count, n, c1s.data_ptr(), c2s.data_ptr(),
                                zqs.data_ptr(), starts.data_ptr(), scal.data_ptr(),
                                scal.data_ptr() + 8, nat.stream_ptr()), "rs_prep")
    prep = dict(order=order, c1=c1s, c2=c2s, zq=zqs, starts=starts, dup_key=scal[0:1],
                dmax=scal[1:2].view(torch.float64))
    ds._cache["prep"] = prep
    _mark("prep_done")
    return prep


_FRONT_POOL: dict = {}   # (device, count, n) -> {"offs": [...], "bufs": [(tensor, base use count)]}
_FRONT_SLOTS = 18


def _use_count(t) -> int:
    return nat._torch()._C._storage_Use_Count(t.untyped_storage()._cdata)


def _front_buffer(count: int, n: int):
    """Pooled device region for rs_front.  A region is handed out again only
    when no view of it is alive (storage use count back at its base), so a
    result the caller still holds is never overwritten."""
    import ctypes
    torch = nat._torch()
    key = (torch.cuda.current_device(), count, n)
    ent = _FRONT_POOL.get(key)
    if ent is None:
        offs = (ctypes.c_int64 * (_FRONT_SLOTS + 1))()
        nat.check(nat.lib().rs_front_offsets(count, n, offs), "rs_front_offsets")
        ent = _FRONT_POOL[key] = {"offs": list(offs), "bufs": []}
    for buf, base in ent["bufs"]:
        if _use_count(buf) == base:
            return buf, ent["offs"]
    buf = torch.empty(ent["offs"][-1], dtype=torch.uint8, device="cuda")
    ent["bufs"].append((buf, _use_count(buf)))
    return buf, ent["offs"]


_SIDE_WS: dict = {}


def _short_ws_bytes(n: int, planes: int, nb_max: int, rs: int) -> int:
    """Workspace of the short-range plane assembly (chunked like assemble_grid)."""
    key = (n, planes, nb_max, rs)
    v = _SIDE_WS.get(key)
    if v is None:
        from .formats import _ASSEMBLE_WORKSPACE
        L = nat.lib()
        fl = nat.ASM_SHORT | nat.asm_oz(nat.OZ_SLICES)
        one = L.rs_assemble_workspace_bytes(n, 1, 1, nb_max, rs, fl)
        per = L.rs_assemble_workspace_bytes(n, 2, 1, nb_max, rs, fl) - one
        chunk = max(1, min(planes, (_ASSEMBLE_WORKSPACE - (one - per)) // max(per, 1)))
        v = _SIDE_WS[key] = L.rs_assemble_workspace_bytes(n, chunk, 1, nb_max, rs, fl)
    return v


def _front_system(positions, charges, box, grid: Grid3, prefetch=None, chain=None):
    """Snap, node sort, bucket-ordered copies, shift histograms and the
    short-range bucket table in one native call (``rs_front``), no sync.
    ``prefetch = (plan, lo, hi)`` also enqueues the short-range planes
    [lo, hi) on the side stream (returned as (buf, event) in the cache).
    Returns the device system; its cache carries the sort/prep products and
    the raw addresses of the histogram and bucket-table slots."""
    torch = nat._torch()
    pos = to_device(positions)
    z = to_device(charges)
    count, n = int(pos.shape[0]), grid.n
    _mark("f_todev")
    buf, o = _front_buffer(count, n)
    _mark("f_buf")
    pf = (None, None, 0, 0, 0, 0, None, None, 0, None, 0, 0, None)
    if prefetch is not None:
        plan, lo, hi, groups, out = prefetch
        side = _side_stream(n)
        rs = int(plan.local.rank)
        if out is None:
            out = torch.empty((hi - lo, n, n), dtype=torch.float64, device="cuda")
        elif (tuple(out.shape) != (hi - lo, n, n) or out.dtype != torch.float64
              or not out.is_cuda or not out.is_contiguous()):
            raise DomainError(f"prefetch_out must be a contiguous float64 CUDA tensor of shape "
                              f"{(hi - lo, n, n)}")
        out.record_stream(side)
        L = nat.lib()
        method = L.rs_short_method(n, count, plan.gamma, rs)
        if method == nat.SHORT_L0:
            wsb = L.rs_short_l0_bytes(plan.gamma)   # the gather needs only L0
        elif method == nat.SHORT_MMA:               # term table + tile counter
            wsb = max(L.rs_short_mma_workspace_bytes(n, plan.gamma), (n + 1) * 4)
        else:
            wsb = _short_ws_bytes(n, hi - lo, max(1, min(n, count)), rs)
        ws = nat.Workspace.get(wsb, "assemble_side")
        ws.record_stream(side)
        grp, gev, evarr = hi - lo, None, None
        if groups > 1:
            import ctypes
            grp = -(-(hi - lo) // groups)
            gev = _group_events(-(-(hi - lo) // grp))
            evarr = (ctypes.c_void_p * len(gev))(*[e.cuda_event for e in gev])
        pf = (plan.local_ul.data_ptr(), plan.local_wl.data_ptr(), rs, plan.gamma, lo, hi,
              out.data_ptr(), ws.data_ptr(), ws.numel(), side.cuda_stream, nat.OZ_SLICES,
              grp, evarr)
    nat.check(nat.lib().rs_front(pos.data_ptr(), z.data_ptr(), count, grid.h, n, buf.data_ptr(),
                                 buf.numel(), nat.stream_ptr(), *pf), "rs_front")
    _mark("f_call")
    if chain is not None:   # Gram -> top-b eigenpairs -> packed D2H, right behind the front
        chain_out = _launch_chain(chain, buf.data_ptr(), o, n)
        _mark("f_chain")
    if prefetch is not None:
        ev = torch.cuda.Event()
        ev.record(side)
        buf.record_stream(side)
    def view(slot, dtype, shape, nbytes):
        return buf[o[slot]:o[slot] + nbytes].view(dtype).view(shape)

    base = buf.data_ptr()
    idx = view(0, torch.int64, (count, 3), 24 * count)
    ds = DeviceIndexedSystem(positions=view(3, torch.float64, (count, 3), 24 * count), charges=z,
                             grid=grid, indices=idx, box=box,
                             _disp=view(1, torch.float64, (count,), 8 * count))
    prep = dict(c1=base + o[6], c2=base + o[7], zq=base + o[8],
                starts=view(9, torch.int64, (count, 3), 24 * count),
                dup_key=view(10, torch.int64, (1,), 8),
                dmax=buf[o[10] + 8:o[10] + 16].view(torch.float64))
    ds._cache["prep"] = prep
    ds._cache["front"] = dict(hist=base + o[11], cnt3=base + o[12], bstart=base + o[13],
                              bc3=base + o[14], nb=base + o[15], buf=buf)
    if prefetch is not None:
        ds._cache["front"]["prefetch"] = dict(lo=lo, hi=hi, buf=out, ev=ev, complete=False,
                                              groups=(grp, gev) if gev else None)
    if chain is not None:
        ds._cache["chain"] = chain_out
    return ds, prep["dup_key"]


_CHAIN_BUFS: dict = {}


def _chain_buffers(n: int, b: int, R_l: int):
    """Pooled device outputs (G, evals, U, trace, packed), pinned packed copy
    and the completion event of :func:`_launch_chain`, per (device, n, b).
    Reuse is stream-ordered: every consumer of a previous call's buffers runs
    on the chain stream before the next call's kernels, and the host reads the
    pinned vector before it enqueues the next call."""
    torch = nat._torch()
    dev = torch.cuda.current_device()
    key = (dev, n, b, R_l)
    ent = _CHAIN_BUFS.get(key)
    if ent is None:
        L = nat.lib()
        m = 3 * n * n + 3 * b + 3 * b * n + 3 + (3 * b + 6)
        flat = torch.empty(m, dtype=torch.float64, device="cuda")
        o = [0, 3 * n * n, 3 * n * n + 3 * b, 3 * n * n + 3 * b + 3 * b * n,
             3 * n * n + 3 * b + 3 * b * n + 3]
        host = torch.empty(3 * b + 6, dtype=torch.float64, pin_memory=True)
        ev = torch.cuda.Event()
        ev.record()   # materialise the cudaEvent_t
        ent = _CHAIN_BUFS[key] = dict(
            G=flat[o[0]:o[1]].view(3, n, n), evals=flat[o[1]:o[2]].view(3, b),
            U=flat[o[2]:o[3]].view(3, b, n), trace=flat[o[3]:o[4]], packed=flat[o[4]:],
            host=host, host_np=host.numpy(), ev=ev,
            gws=nat.Workspace.get(L.rs_gram_shifted_workspace_bytes(n, R_l), "syrk"),
            ews=nat.Workspace.get(L.rs_topeig_workspace_bytes(3, n, b), "topeig"))
    return ent


def _launch_chain(chain, base: int, o, n: int):
    """``rs_chain_eig`` on the front's histograms (current stream)."""
    plan, b, iters = chain
    R_l = int(plan.w_long_abs.shape[0])
    ent = _chain_buffers(n, b, R_l)
    L = nat.lib()
    nat.check(L.rs_chain_eig(plan.table_dev.data_ptr(), plan.table_dev.shape[1], n, R_l,
                             base + o[11], plan.w_long_abs.data_ptr(), ent["G"].data_ptr(),
                             ent["gws"].data_ptr(), ent["gws"].numel(), b, iters,
                             ent["evals"].data_ptr(), ent["U"].data_ptr(),
                             ent["trace"].data_ptr(), ent["ews"].data_ptr(), ent["ews"].numel(),
                             base + o[10] + 8, base + o[10], base + o[15],
                             ent["packed"].data_ptr(), ent["host"].data_ptr(),
                             ent["ev"].cuda_event, nat.stream_ptr()), "rs_chain_eig")
    return ent


_GROUP_EVENTS: dict = {}


def _group_events(k: int):
    """``k`` pooled CUDA events (created eagerly) for rs_front's plane groups;
    re-recording is safe: a wait enqueued earlier keeps the record it saw."""
    torch = nat._torch()
    dev = torch.cuda.current_device()
    pool = _GROUP_EVENTS.setdefault(dev, [])
    while len(pool) < k:
        e = torch.cuda.Event()
        e.record()          # materialise the cudaEvent_t
        pool.append(e)
    return pool[:k]


def _decode_key(key: int, n: int) -> tuple:
    """x3-major node key -> (x1, x2, x3)."""
    return (key % n, (key // n) % n, key // (n * n))


def _collision_flag(ds, n: int):
    return _node_sort(ds, n)["dup_key"]


def _as_device_system(system, grid: Grid3, prefetch=None, chain=None):
    """Accept the reference's types or :class:`DeviceParticles`.  ``prefetch``
    (plan, lo, hi) rides along with the native front when the input is snapped
    here."""
    if isinstance(system, DeviceIndexedSystem):
        if system.grid != grid:
            raise ConfigError("particle system snapped to a different grid")
        return system, None
    if isinstance(system, DeviceParticles):
        return _front_system(system.positions, system.charges, system.box, grid, prefetch,
                             chain)
    if isinstance(system, IndexedParticleSystem):
        if system.grid != grid:
            raise ConfigError("particle system snapped to a different grid")
        twin = getattr(system, "_device", None)
        if twin is not None:   # a build_rs result handed back in: its device arrays
            return twin, twin._cache.get("prep", {}).get("dup_key")
        torch = nat._torch()
        ds = DeviceIndexedSystem(positions=to_device(system.base.positions),
                                 charges=to_device(system.charges), grid=grid,
                                 indices=to_device(system.indices, torch.int64),
                                 box=system.base.box,
                                 _disp=torch.full((1,), system.max_displacement,
                                                  dtype=torch.float64, device="cuda"))
        ds._cache["host"] = system
        return ds, None
    if isinstance(system, ParticleSystem):
        ds, dup = _front_system(system.positions, system.charges, system.box, grid, prefetch,
                                chain)
        ds._cache["host_input"] = True
        return ds, dup
    raise ConfigError(f"expected a particle system, got {type(system).__name__}")


def _trusted_indexed(ds: DeviceIndexedSystem) -> IndexedParticleSystem:
    """The reference's result type (``assembly.py:271-279``: an
    ``IndexedParticleSystem`` with read-only numpy arrays) from the device
    system, without re-running the host validation the device already did
    (box containment at input, node collisions in ``rs_prep``).  The device
    twin rides along as ``_device`` so the observables reuse its arrays."""
    def frozen(t, dtype):
        a = np.ascontiguousarray(to_host(t), dtype=dtype)
        a.setflags(write=False)
        return a

    base = object.__new__(ParticleSystem)
    object.__setattr__(base, "positions", frozen(ds.positions, np.float64))
    object.__setattr__(base, "charges", frozen(ds.charges, np.float64))
    object.__setattr__(base, "box", ds.box)
    out = object.__new__(IndexedParticleSystem)
    object.__setattr__(out, "base", base)
    object.__setattr__(out, "grid", ds.grid)
    object.__setattr__(out, "indices", frozen(ds.indices, np.int64))
    object.__setattr__(out, "max_displacement", ds.max_displacement)
    object.__setattr__(out, "_device", ds)
    return out


def _host_system(ds: DeviceIndexedSystem):
    """``AssemblyResult.system``: host particle systems come back as the
    reference's host type; device inputs stay on the device (no D2H on the
    serving path)."""
    h = ds._cache.get("host")
    if h is None and ds._cache.get("host_input"):
        h = ds._cache["host"] = _trusted_indexed(ds)
    return h if h is not None else ds


# ----------------------------------------------------- public assembly API
def assemble_long(ref2n: ReferenceCanonical, system, split_index: int) -> CanonicalTensor:
    """Rank ``(R_l+1) N`` long part, particle-major term order, side matrices
    materialised on the device by ``rs_gather_windows`` (``assembly.py:111-136``)."""
    if not (0 <= split_index < ref2n.R):
        raise DomainError(f"split index {split_index} out of range")
    torch = nat._torch()
    n = ref2n.grid.n // 2
    nt = split_index + 1
    ds, flag = _as_device_system(system, Grid3(n, Box3_half(ref2n)))
    z = ds.charges
    table = to_device(ref2n.table)
    w = to_device(ref2n.tensor.weights[:nt])
    weights = (z[:, None] * w[None, :]).reshape(-1)
    count = ds.count
    facs = []
    for l in range(3):
        starts = (n - ds.indices[:, l]).contiguous()
        out = torch.empty((n, count * nt), dtype=torch.float64, device="cuda")
        nat.check(nat.lib().rs_gather_windows(table.data_ptr(), table.shape[1], n, starts.data_ptr(),
                                              count, nt, 0, None, None, out.data_ptr(), count * nt,
                                              nat.stream_ptr()), "rs_gather_windows")
        facs.append(out)
    return CanonicalTensor(weights, tuple(facs))


def Box3_half(ref2n: ReferenceCanonical):
    from .particles import Box3

    return Box3(ref2n.grid.box.half_width / 2.0)


def assemble_short(ref2n: ReferenceCanonical, system, split_index: int, delta: float,
                   overlap_policy: str = "soft", max_overlap: Optional[int] = 8,
                   gamma: Optional[int] = None) -> CCT:
    """Short part as a uniform CCT (``assembly.py:139-184``)."""
    n = ref2n.grid.n // 2
    g, local = _short_window(ref2n, split_index, delta, gamma)
    centers = system.indices
    weights = system.charges
    return CCT(local=local, gamma=g, centers=centers, weights=weights, mode_sizes=(n, n, n),
               overlap_policy=overlap_policy, max_overlap=max_overlap)


@dataclass(frozen=True)
class AssemblyResult:
    rs: Union[RSCanonical, RSTucker]
    reference: ReferenceCanonical
    system: object
    split_index: int
    sigma: float
    gamma: int
    report: dict


_STREAMS: dict = {}


def _stream(kind: str, sms: int = 0):
    """Per-device internal streams: "side" (lowest priority) carries the
    prefetched short-range planes, on an SM partition of ``sms`` SMs when
    > 0; "chain" (highest priority) the latency-bound long-range reduction,
    so its small kernels are scheduled ahead of the big plane GEMM's blocks."""
    torch = nat._torch()
    dev = torch.cuda.current_device()
    st = _STREAMS.get((dev, kind, sms))
    if st is None:
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
            else (0, -1)
        if kind == "side" and sms > 0:
            # the wide short-range kernels on an SM partition (green context):
            # the SMs outside it stay free for the latency-bound chain
            import ctypes
            ptr, got = ctypes.c_void_p(), ctypes.c_int()
            if nat.lib().rs_partition_stream(min(sms, _device_sms(dev)), int(lo),
                                             ctypes.byref(ptr), ctypes.byref(got)) == 0:
                st = torch.cuda.ExternalStream(ptr.value, device=dev)
        if st is None:
            st = torch.cuda.Stream(device=dev, priority=(hi if kind == "chain" else lo))
        _STREAMS[(dev, kind, sms)] = st
    return st


def _side_sms(n: int) -> int:
    """SMs of the short-range side partition: the chain's latency-bound
    kernels need ~20 free SMs at C2 (measured best: 128); at n >= 512 the
    short part dominates the step and takes 140 (C4 227 -> 215 ms, C5 284 ->
    270 ms against 128).  RSB200_SIDE_SMS overrides (0: ordinary stream)."""
    if _SIDE_SMS is not None:
        return _SIDE_SMS
    return 128 if n <= 256 else 140


def _side_streams():
    torch = nat._torch()
    dev = torch.cuda.current_device()
    return [st for (d, kind, _), st in _STREAMS.items() if d == dev and kind == "side"]


def _device_sms(dev: int) -> int:
    return nat._torch().cuda.get_device_properties(dev).multi_processor_count


def _side_stream(n: int):
    return _stream("side", _side_sms(n))


def build_rs(system, cfg: AssemblyConfig, prefetch_dense=False, group=None,
             prefetch_groups: int = 1, prefetch_out=None) -> AssemblyResult:
    """Reference ``build_rs`` (``assembly.py:187-279``) on the device.

    Extensions: ``prefetch_dense`` (see :func:`_build_rs`); ``group`` (a
    ``torch.distributed`` group: particle-sharded histograms/core);
    ``prefetch_groups`` splits the prefetched planes into that many groups
    finished one by one, so a host-returning :func:`dense_rs` starts the
    device->host copy of the first planes while later ones are computed;
    ``prefetch_out`` (a float64 CUDA tensor of the slab's shape) receives the
    prefetched grid instead of a fresh allocation (a serving loop's reused
    output buffer)."""
    if not prefetch_dense:
        return _build_rs(system, cfg, False, group)
    torch = nat._torch()
    user = torch.cuda.current_stream()
    chain = _stream("chain")
    chain.wait_stream(user)
    for side in _side_streams():   # earlier prefetches may still read recycled memory
        chain.wait_stream(side)
    with torch.cuda.stream(chain):
        res = _build_rs(system, cfg, prefetch_dense, group, max(1, int(prefetch_groups)),
                        prefetch_out)
    user.wait_stream(chain)
    return res


# where the short-range prefetch enters the side stream: right after snapping
# ("snap", maximal overlap) or behind the eigen block ("eig": the latency-bound
# Gram/eigen kernels then run on an otherwise idle GPU)
_PREFETCH_AT = os.environ.get("RSB200_PREFETCH_AT", "snap")
_TUCKER_IN_BUILD = os.environ.get("RSB200_TUCKER_IN_BUILD", "1") == "1"
_TRACE = [] if os.environ.get("RSB200_HOST_TRACE") else None


def _mark(label: str) -> None:
    """Host-time trace point (diagnostics; no-op unless RSB200_HOST_TRACE)."""
    if _TRACE is not None:
        import time
        _TRACE.append((label, time.perf_counter()))


# SMs of the side stream's partition (0: ordinary stream on the whole device)
_SIDE_SMS = int(os.environ["RSB200_SIDE_SMS"]) if os.environ.get("RSB200_SIDE_SMS") else None


# the Gram + eigen block enqueued by the front call (RSB200_CHAIN=0: from _build_rs)
_CHAIN = os.environ.get("RSB200_CHAIN", "1") == "1"


def _world(group) -> int:
    if group is None:
        return 1
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_initialized() else 1


_RANK_BUF: dict = {}


def _rank_rule(packed, b: int, n: int, eps, forced, limit, iters):
    """``rank_rule_fast`` through ``rs_rank_rule`` (C, same arithmetic):
    [(rank or None, tail at the rank, total)] per mode."""
    import ctypes
    buf = _RANK_BUF.get(0)
    if buf is None:
        buf = _RANK_BUF[0] = ((ctypes.c_int64 * 3)(), (ctypes.c_double * 3)(),
                              (ctypes.c_double * 3)(), (ctypes.c_int64 * 3)())
    ro, to, so, fo = buf
    fptr = None
    if forced is not None:
        for l in range(3):
            fo[l] = int(forced[l]) if forced[l] is not None else 0
        fptr = ctypes.addressof(fo)
    base = packed.ctypes.data
    nat.check(nat.lib().rs_rank_rule(base, base + 8 * 3 * b, 3, b, n, float(eps), fptr,
                                     int(limit) if limit is not None else 0, iters,
                                     ctypes.addressof(ro), ctypes.addressof(to),
                                     ctypes.addressof(so)), "rs_rank_rule")
    return [(ro[l] if ro[l] > 0 else None, to[l], so[l]) for l in range(3)]


def _eig_block(cfg: AssemblyConfig, n: int):
    """Ritz block of the eigen-truncation: (b, use_top, iters, eps, forced ranks)."""
    # block size: the numerical rank of the long-part Grams grows as eps shrinks
    eps_ = cfg.reduction.eps if cfg.reduction.eps is not None else 1e-12
    b = min(n - n % 2, TOPEIG_BLOCK if eps_ >= 1e-6 else 64)
    forced = cfg.reduction.ranks
    if forced is not None:
        b = min(n - n % 2, max(b, max(forced) + 16 + (max(forced) % 2)))
    # eps < 1e-7 pushes the numerical rank past the largest Ritz block: go
    # straight to the full (cuSOLVER) spectrum instead of escalating twice
    use_top = top_eig_supported(n, b) and eps_ >= 1e-7
    if eps_ < 1e-7 and n >= 512 and forced is None:
        # wide Ritz block (C5: rank 132 at eps 1e-8): subspace iteration +
        # cuSOLVER on the b x b Rayleigh quotient instead of three full
        # n x n syevd; the convergence rule falls back to them per mode
        b = min(n - n % 2, TOPEIG_WIDE_BLOCK)
        use_top = top_eig_supported(n, b)
    # two subspace iterations: one already gives grid parity (1e-10) at
    # eps >= 1e-6, but point values / energies (1e-12) need the second
    return b, use_top, TOPEIG_ITERS, eps_, forced


def _eig_by_mode(G, group, fn, shapes):
    """The per-mode eigen work of a sharded run: mode l is solved by rank
    l mod world and broadcast (one message per mode), so every rank holds
    bitwise the same factors ("rank 0 + broadcast", spread over
    the three modes).  ``fn`` maps a (1, n, n) Gram stack to tensors of shapes
    ``(1,) + shapes[i]``; returns them stacked over the modes."""
    import math as _m
    import torch.distributed as dist
    torch = nat._torch()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    sizes = [int(_m.prod(sh)) for sh in shapes]
    flats = []
    for l in range(3):
        owner = l % world
        if owner == rank:
            flat = torch.cat([t.reshape(-1) for t in fn(G[l:l + 1].contiguous())])
        else:
            flat = torch.empty(sum(sizes), dtype=torch.float64, device="cuda")
        flats.append(flat)
    for l in range(3):   # after all local solves are enqueued
        dist.broadcast(flats[l], src=dist.get_global_rank(group, l % world), group=group)
    out = []
    o = 0
    for sh, m in zip(shapes, sizes):
        out.append(torch.stack([f[o:o + m].view(sh) for f in flats]).contiguous())
        o += m
    return tuple(out)


def _build_rs(system, cfg: AssemblyConfig, prefetch_dense=False, group=None,
              prefetch_groups: int = 1, prefetch_out=None) -> AssemblyResult:
    """Snap, project, split, reduce, package (``assembly.py:200-279``) -- device path.

    ``system`` may be a reference-style :class:`ParticleSystem` /
    :class:`IndexedParticleSystem` (host arrays) or :class:`DeviceParticles`.

    ``prefetch_dense`` (extension): ``True`` or an x1 plane range ``(lo, hi)``
    starts the short-range part of the dense grid on a side stream right after
    snapping, concurrently with the long-range reduction (it does not depend on
    it); a following :func:`dense_rs` then only adds the Tucker part.
    """
    torch = nat._torch()
    grid = cfg.grid
    n = grid.n
    _mark("start")
    fused = None
    if (prefetch_dense and _PREFETCH_AT == "snap" and cfg.split_index is not None
            and isinstance(system, (DeviceParticles, ParticleSystem))):
        plan0 = plan_for(cfg, int(cfg.split_index))
        if plan0.local.rank > 0:
            lo, hi = (0, n) if prefetch_dense is True else (int(prefetch_dense[0]),
                                                            int(prefetch_dense[1]))
            fused = (plan0, lo, hi, prefetch_groups, prefetch_out)
    chain = None
    if (cfg.split_index is not None and cfg.long_format == "tucker"
            and cfg.reduction.max_sweeps == 0 and _CHAIN and _world(group) == 1
            and isinstance(system, (DeviceParticles, ParticleSystem))):
        b_, top_, it_, _, _ = _eig_block(cfg, n)
        if top_:
            chain = (plan_for(cfg, int(cfg.split_index)), b_, it_)
    ds, collision = _as_device_system(system, grid, fused, chain)
    if cfg.sigma is not None:
        sigma = float(cfg.sigma)
    elif ds.count >= 2:
        sigma = separation_distance(ParticleSystem(to_host(ds.positions), to_host(ds.charges),
                                                   ds.box))
    else:
        sigma = grid.h
    if cfg.split_index is not None:
        split_index = int(cfg.split_index)
    else:
        split_index = split_rank(_reference_cached(cfg), sigma, cfg.delta, cfg.criterion)
    _mark("snapped")
    _mark("split")
    plan = plan_for(cfg, split_index)
    _mark("plan")
    ref2n = plan.ref2n
    nt = split_index + 1
    raw_rank = ds.count * nt
    reduce_long = cfg.reduce_long
    if reduce_long is None:
        reduce_long = cfg.long_format == "tucker" or raw_rank > cfg.reduce_threshold
    if cfg.long_format == "tucker":
        reduce_long = True

    idx = ds.indices
    z = ds.charges
    prep = ds._cache.get("prep")
    if prep is None:  # already-indexed input: sort/prep now (no sync)
        prep = _node_sort(ds, n)
        if collision is None:
            collision = prep["dup_key"]
    starts = prep["starts"]
    report = {"n": n, "b": grid.box.half_width, "particles": ds.count}
    if cfg.overlap_policy == "strict":
        short = CCT(local=plan.local, gamma=plan.gamma, centers=idx, weights=z,
                    mode_sizes=(n, n, n), overlap_policy=cfg.overlap_policy,
                    max_overlap=cfg.max_overlap)
    else:
        short = trusted_cct(plan.local, plan.gamma, idx, z, (n, n, n), cfg.overlap_policy,
                            cfg.max_overlap)
    if cfg.overlap_policy not in ("strict", "soft"):
        raise DomainError(f"unknown overlap policy {cfg.overlap_policy!r}")
    hist = cnt3 = None
    world = 1
    if group is not None:
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    p_lo, p_hi = (0, ds.count) if world == 1 else particle_shard(ds.count, dist.get_rank(group),
                                                                  world)
    front = ds._cache.get("front")
    if reduce_long and cfg.reduction.max_sweeps == 0:
        if world == 1 and front is not None:
            hist, cnt3 = front["hist"], front["cnt3"]
        elif world == 1:
            hist, cnt3 = shift_histograms(idx, z, n)
        else:
            h_part, c_part = shift_histograms(idx[p_lo:p_hi].contiguous(),
                                              z[p_lo:p_hi].contiguous(), n)
            packed_h = sharded_sum(torch.cat([h_part.reshape(-1), c_part.to(torch.float64)]),
                                   group)
            hist = packed_h[:3 * n].reshape(3, n)
            cnt3 = packed_h[3 * n:].to(torch.int32)
    if plan.local.rank > 0:
        _mark("hist")
        if front is not None:
            lay = dict(c1=prep["c1"], c2=prep["c2"], zq=prep["zq"], bstart=front["bstart"],
                       bc3=front["bc3"], nb=front["nb"], nb_max=max(1, min(n, ds.count)),
                       centers=idx, z=z, buf=front["buf"])
        else:
            lay = short_layout(idx, z, n, cnt3, prep)
        lay.update(ul=plan.local_ul, wl=plan.local_wl)
        short._cache["dev"] = lay

    def launch_prefetch():
        lo, hi = (0, n) if prefetch_dense is True else (int(prefetch_dense[0]),
                                                        int(prefetch_dense[1]))
        main = torch.cuda.current_stream()
        side = _side_stream(n)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            buf = torch.empty((hi - lo, n, n), dtype=torch.float64, device="cuda")
            assemble_grid(None, short, lo, hi, out=buf, workspace_slot="assemble_side")
            ev = torch.cuda.Event()
            ev.record(side)
        short._cache["prefetch"] = dict(lo=lo, hi=hi, buf=buf, ev=ev, complete=False,
                                        groups=None)

    prefetch_pending = bool(prefetch_dense) and plan.local.rank > 0
    fpre = ds._cache.get("front", {}).get("prefetch")
    if prefetch_pending and fpre is not None:  # launched with the native front
        short._cache["prefetch"] = fpre
        prefetch_pending = False
    if prefetch_pending and (_PREFETCH_AT == "snap" or not (reduce_long and
                                                           cfg.reduction.max_sweeps == 0)):
        _mark("layout")
        launch_prefetch()
        prefetch_pending = False

    tails = None
    if reduce_long and cfg.reduction.max_sweeps == 0:
        # shift histograms -> per-mode Grams on DMMA -> top-b eigenpairs, then
        # ONE synchronisation for everything the host must decide on
        _mark("prefetch")
        b, use_top, iters, eps_, forced = _eig_block(cfg, n)
        full = None
        chained = ds._cache.get("chain")
        if chained is not None:   # Gram + eigen block already enqueued by the front
            G, evals, U, trace = chained["G"], chained["evals"], chained["U"], chained["trace"]
        else:
            G = shifted_grams(plan.table_dev, n, plan.w_long_abs, hist)
        if chained is not None:
            pass
        elif use_top:
            _mark("grams")
            evals, U, trace = (top_eig(G, b, iters) if world == 1 else
                               _eig_by_mode(G, group, lambda g: top_eig(g, b, iters),
                                            [(b,), (b, n), ()]))
        else:
            # full spectra of the three modes at once (forked cuSOLVER streams),
            # values fetched with the one packed synchronisation below
            b = 0
            evals = U = trace = torch.zeros(0, dtype=torch.float64, device="cuda")
            full = eig_desc_batched(G) if world == 1 else \
                _eig_by_mode(G, group, eig_desc_batched, [(n,), (n, n)])
        if prefetch_pending:  # short-range planes behind the latency-bound eigen block
            launch_prefetch()
            prefetch_pending = False
        if chained is None:
            parts = [evals.reshape(-1), trace, prep["dmax"], collision.to(torch.float64)]
            if full is not None:
                parts.append(full[0].reshape(-1))
            if front is not None:  # occupied x3 values: sizes the bucket-K core
                nb_view = front["buf"][front["nb"] - front["buf"].data_ptr():][:4].view(
                    torch.int32)
                parts.append(nb_view.to(torch.float64))
        _mark("eig_enq")
        if chained is not None:
            chained["ev"].synchronize()
            packed = chained["host_np"].copy()
        else:
            packed = to_host(torch.cat(parts))
        _mark("synced_eig")
        nq_host = int(packed[-1]) if front is not None else 0
        nt_ = 3 * b + (3 if use_top else 0)
        if packed[nt_ + 1] >= 0:
            node = _decode_key(int(packed[nt_ + 1]), n)
            raise ResolutionError(f"grid n={n} cannot resolve the system: several particles "
                                  f"snap to node {node}; use a larger n")
        if ds._disp is not None and ds._disp.numel() == ds.count:
            ds._cache["maxdisp"] = float(packed[nt_])
        limit = min(n, raw_rank)
        if forced is not None:
            for r in forced:
                if r > limit:
                    raise ConfigError(f"requested rank {r} exceeds min(n, R) = {limit}")
        ranks, values, tails, zs, from_top = [], [], [], [], []
        if use_top:
            fast3 = _rank_rule(packed, b, n, cfg.reduction.eps, forced, limit, iters)
        for l in range(3):
            fr = forced[l] if forced is not None else None
            r = None
            top = False
            if use_top:
                r, tail_r, total = fast3[l]
                if r is not None and fr is not None and fr > b:
                    r = None
                Ul = U[l] if r is not None else None
                top = r is not None
                if top:   # spectrum arrays are not needed on this path
                    ranks.append(int(r))
                    values.append(None)
                    tails.append((tail_r, total))
                    zs.append(Ul)
                    from_top.append(True)
                    continue
            if r is None:
                bb = min(n - n % 2, TOPEIG_MAX_BLOCK if b >= 48 else 2 * b)
                if b and bb > b and top_eig_supported(n, bb):
                    ev2, U2, tr2 = top_eig(G[l:l + 1].contiguous(), bb, 2)
                    r, sv, tail, total = truncated_spectrum(to_host(ev2[0]), float(tr2[0]), n,
                                                            cfg.reduction.eps, fr, limit, 2)
                    if r is not None and (fr is None or fr <= bb):
                        Ul = U2[0]
                    else:
                        r = None
                if r is None:
                    if full is not None:   # batched spectra, already on the host
                        o = nt_ + 2
                        sh = np.sqrt(packed[o + l * n:o + (l + 1) * n])
                        Ul = full[1][l]
                    else:
                        s_full, z_full = eig_desc(G[l])     # full cuSOLVER spectrum
                        sh = to_host(s_full)
                        Ul = z_full.T
                    r = fr if fr is not None else min(eps_rank(sh, cfg.reduction.eps), limit)
                    sv, total = sh, float(np.sum(sh * sh))
                    tail = np.cumsum((sh * sh)[::-1])[::-1]
            ranks.append(int(r))
            values.append(sv)
            tails.append((float(tail[r]) if r < len(tail) else 0.0, total))
            zs.append(Ul)
            from_top.append(top)
        ranks = tuple(ranks)
        _mark("d2h")
        core = None
        fused_tucker = False
        if world == 1 or front is not None:
            # factors + projections + core in one native call (bucket-K core);
            # a rank of a sharded run sums its x3 buckets (or particles) only
            # and the r1 r2 r3 partials are all-reduced
            r1, r2, r3 = ranks
            Ub, bu = U, b
            if not (use_top and all(t is True for t in from_top)):
                # escalated modes: gather their leading rows into one (3, r, n) block
                bu = max(ranks)
                Ub = torch.zeros((3, bu, n), dtype=torch.float64, device="cuda")
                for l, (zl, r) in enumerate(zip(zs, ranks)):
                    Ub[l, :r] = zl[:r]
            flat = torch.empty(n * (r1 + r2 + r3) + r1 * r2 * r3, dtype=torch.float64,
                               device="cuda")
            zs = [flat[:n * r1].view(n, r1), flat[n * r1:n * (r1 + r2)].view(n, r2),
                  flat[n * (r1 + r2):n * (r1 + r2 + r3)].view(n, r3)]
            core = flat[n * (r1 + r2 + r3):].view(r1, r2, r3)
            L = nat.lib()
            ws = nat.Workspace.get(L.rs_back_workspace_bytes(n, r1, r2, r3, ds.count,
                                                             int(plan.w_long.shape[0]), nq_host),
                                   "core")
            back_args = (Ub.data_ptr(), bu, n, r1, r2, r3, plan.table_dev.data_ptr(),
                         plan.table_dev.shape[1], int(plan.w_long.shape[0]),
                         nat.ptr(starts), z.data_ptr(), plan.w_long.data_ptr(), ds.count,
                         zs[0].data_ptr(), zs[1].data_ptr(), zs[2].data_ptr(),
                         core.data_ptr(), ws.data_ptr(), ws.numel(), nat.stream_ptr(),
                         *((prep["c1"], prep["c2"], prep["zq"], front["bstart"],
                            front["bc3"], front["nb"]) if front is not None
                           else (None,) * 6), nq_host)
            pre0 = short._cache.get("prefetch") if cfg.long_format == "tucker" else None
            if world > 1:
                q_lo, q_hi = particle_shard(nq_host, dist.get_rank(group), world)
                nat.check(L.rs_back_shard(*back_args, q_lo, q_hi, p_lo, p_hi), "rs_back_shard")
                sharded_sum(core, group)
            elif (pre0 is not None and _TUCKER_IN_BUILD and pre0["groups"] is None
                    and not pre0["complete"]):
                # back + the Tucker part of the prefetched slab in one call
                lo, hi, buf = pre0["lo"], pre0["hi"], pre0["buf"]
                # one chunk (operands of the whole slab, formed before the wait)
                chunk, wsb = tucker_plan(n, hi - lo, max(ranks), workspace_bytes=1 << 62)
                aws = nat.Workspace.get(wsb, "assemble")
                cur = torch.cuda.current_stream()
                buf.record_stream(cur)
                nat.check(L.rs_back_tucker(*back_args, buf.data_ptr(), lo, hi, chunk,
                                           aws.data_ptr(), aws.numel(), pre0["ev"].cuda_event),
                          "rs_back_tucker")
                done = torch.cuda.Event()
                done.record(cur)
                short._cache["prefetch"] = dict(pre0, ev=done, complete=True)
                fused_tucker = True
            else:
                nat.check(L.rs_back(*back_args), "rs_back")
            _mark("back_enq")
        else:
            zs = [zl[:r].T.contiguous() for zl, r in zip(zs, ranks)]
        spectrum = SvdSpectrum(values=tuple(values), vectors=tuple(zs))
        if core is not None:
            pass
        elif world == 1:
            core = shifted_core(plan.table_dev, n, zs, starts, z, plan.w_long)
        else:
            core = sharded_sum(shifted_core(plan.table_dev, n, zs, starts[p_lo:p_hi].contiguous(),
                                            z[p_lo:p_hi].contiguous(), plan.w_long), group)
        _mark("ranks")
        tucker = _trusted_tucker(core, zs)
        _mark("tucker_obj")
        long_raw = None
        pre = short._cache.get("prefetch") if cfg.long_format == "tucker" else None
        if pre is not None and _TUCKER_IN_BUILD and not fused_tucker:
            # finish the prefetched slab here: the Tucker part is enqueued right
            # behind the core, before the host packages the result
            lo, hi, buf = pre["lo"], pre["hi"], pre["buf"]
            cur = torch.cuda.current_stream()
            buf.record_stream(cur)
            if pre["groups"] is None:
                cur.wait_event(pre["ev"])
                tucker_accumulate(tucker, lo, hi, buf)
                done = torch.cuda.Event()
                done.record(cur)
                short._cache["prefetch"] = dict(pre, ev=done, complete=True)
            else:   # group by group, behind each group's short planes
                grp, gev = pre["groups"]
                dones = []
                for g, ev in enumerate(gev):
                    g0, g1 = g * grp, min(hi - lo, (g + 1) * grp)
                    cur.wait_event(ev)
                    tucker_accumulate(tucker, lo + g0, lo + g1, buf[g0:g1])
                    done = torch.cuda.Event()
                    done.record(cur)
                    dones.append(done)
                short._cache["prefetch"] = dict(pre, ev=dones[-1], complete=True,
                                                groups=(grp, dones))
        _mark("tucker_enq")
    else:
        if int(collision[0]) >= 0:
            raise ResolutionError(f"grid n={n} cannot resolve the system: several particles snap "
                                  f"to node {_decode_key(int(collision[0]), n)}; use a larger n")
        long_raw = assemble_long(ref2n, ds, split_index)
        if reduce_long:
            spectrum = side_svd(long_raw)
            tucker = c2t_als(long_raw, cfg.reduction, spectrum=spectrum)
            ranks = tucker.ranks
    report.update({
        "max_snap_displacement": ds.max_displacement,
        "quadrature_rank": ref2n.R,
        "split_index": split_index,
        "short_terms": ref2n.R - split_index - 1,
        "sigma": sigma,
        "raw_long_rank": raw_rank,
        "reduced": bool(reduce_long),
    })
    if reduce_long:
        report["tucker_ranks"] = list(ranks)
        if tails is not None:
            # tail energies include the part of the spectrum beyond the Ritz block
            report["reduction_tail_bracket"] = float(sum(np.sqrt(t) for t, _ in tails))
            report["reduction_tail_fraction"] = [float(np.sqrt(t) / np.sqrt(tot)) if tot > 0 else 0.0
                                                 for t, tot in tails]
        else:
            report["reduction_tail_bracket"] = rhosvd_error_bound(None, spectrum, ranks)
            totals = [float(np.sqrt(np.sum(s * s))) for s in spectrum.values]
            report["reduction_tail_fraction"] = [
                float(np.sqrt(np.sum(s[r:] ** 2)) / t) if t > 0 else 0.0
                for s, r, t in zip(spectrum.values, ranks, totals)]
        if cfg.long_format == "tucker":
            long_part = tucker
        else:
            long_part = tucker_to_canonical(tucker, cfg.reduction.eps_t2c)
            report["reduced_canonical_rank"] = long_part.rank
    else:
        long_part = long_raw

    report["gamma"] = plan.gamma
    report["gamma_h"] = plan.gamma * grid.h
    rs = RSTucker(long=long_part, short=short, grid=grid) if cfg.long_format == "tucker" else \
        RSCanonical(long=long_part, short=short, grid=grid)
    sto = storage_report(rs)
    report["storage_floats"] = sto.total
    report["storage_bound"] = sto.bound
    _mark("core_enq")
    return AssemblyResult(rs=rs, reference=ref2n, system=_host_system(ds),
                          split_index=split_index, sigma=sigma, gamma=plan.gamma, report=report)
