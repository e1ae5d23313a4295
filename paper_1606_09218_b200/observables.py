"""Energies and forces from the RS representation, on the device.

Reference: ``observables.py``.  The tensor energy uses the long part only,
``E = 1/2 sum_j z_j (P_l(x_j)/h^3 - z_j P_Rl(0))`` (``observables.py:101-129``);
``reference_energy`` / ``force_fd`` are the O(N^2 R_l) windowed direct sums
over the unreduced long part (``:190-259``).  Every reduction the reference
does with ``math.fsum`` is done here in double-double with a fixed order
(``rs_sum_dd``, ``rs_pair_sums``), so results agree with the exactly
rounded reference sums to within the rounding of the individual terms.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as nat
from .errors import ConfigError, DomainError, SeparationError, SingularityError
from .formats import CanonicalTensor, RSCanonical, RSTucker, TuckerTensor, eval_canonical_many, \
    eval_tucker_many, to_device, to_host
from .particles import ParticleSystem, separation_distance


@dataclass(frozen=True)
class EnergyReport:
    energy: float
    exact: Optional[float] = None
    abs_error: Optional[float] = None
    rel_error: Optional[float] = None
    flagged: bool = False
    timings: dict = field(default_factory=dict)

    @classmethod
    def with_oracle(cls, energy: float, exact: float, flagged: bool = False, timings=None):
        err = abs(energy - exact)
        rel = err / abs(exact) if exact != 0 else math.inf
        return cls(energy=energy, exact=exact, abs_error=err, rel_error=rel, flagged=flagged,
                   timings=timings or {})


@dataclass(frozen=True)
class ForceVector:
    index: int
    force: np.ndarray

    def __post_init__(self):
        f = np.asarray(self.force, dtype=np.float64).reshape(3)
        if not np.all(np.isfinite(f)):
            raise DomainError(f"non-finite force on particle {self.index}")
        object.__setattr__(self, "force", f)


def dd_sum(v) -> float:
    """Compensated fixed-order device sum of a 1-D CUDA tensor (``rs_sum_dd``)."""
    torch = nat._torch()
    v = v.contiguous()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L = nat.lib()
    ws = nat.Workspace.get(L.rs_sum_workspace_bytes(v.numel()), "sum")
    nat.check(L.rs_sum_dd(v.data_ptr(), v.numel(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                          nat.stream_ptr()), "rs_sum_dd")
    return out


def _long_values(rs, indices):
    if isinstance(rs, RSCanonical):
        return eval_canonical_many(rs.long, indices, device=True)
    if isinstance(rs, RSTucker):
        return eval_tucker_many(rs.long, indices, device=True)
    if isinstance(rs, CanonicalTensor):
        return eval_canonical_many(rs, indices, device=True)
    if isinstance(rs, TuckerTensor):
        return eval_tucker_many(rs, indices, device=True)
    raise ConfigError(f"cannot evaluate a long part of type {type(rs).__name__}")


def _system_arrays(system):
    torch = nat._torch()
    system = getattr(system, "_device", system)   # host result of build_rs: its device twin
    return to_device(system.indices, torch.int64), to_device(system.charges)


def particle_potentials(rs, system, reference, device: bool = False):
    """Per-particle long-range potential ``phi_j = P_l(x_j)/h^3 - z_j P_Rl(0)``
    (the ``rs_energy`` summand divided by ``z_j``)."""
    if reference.split_index is None:
        raise ConfigError("reference carries no split index")
    idx, z = _system_arrays(system)
    h3 = system.grid.h ** 3
    phi = _long_values(rs, idx) / h3 - z * reference.self_value()
    return phi if device else to_host(phi)


def rs_energy(rs, system, reference, check_separation: bool = True) -> float:
    """Long-part interaction energy (``observables.py:101-129``)."""
    if reference.split_index is None:
        raise ConfigError("reference carries no split index")
    gamma = getattr(getattr(rs, "short", None), "gamma", None)
    if check_separation and gamma is not None and system.count >= 2 and \
            getattr(rs.short.local, "rank", 0) > 0:
        support = gamma * system.grid.h
        base = system.base
        sep = separation_distance(base if isinstance(base, ParticleSystem) else
                                  ParticleSystem(to_host(system.positions),
                                                 to_host(system.charges), system.box))
        if support >= sep:
            warnings.warn(f"short-range support {support:.3g} reaches the separation distance "
                          f"{sep:.3g}; the energy cancellation is degraded", stacklevel=2)
    idx, z = _system_arrays(system)
    h3 = system.grid.h ** 3
    values = _long_values(rs, idx) / h3
    terms = z * (values - z * reference.self_value())
    return 0.5 * float(dd_sum(terms))


def _fd_rows(u, h: float):
    """Central differences inside, one-sided at the two ends, on every column
    (``observables.py:132-139``); device tensor in, device tensor out."""
    out = torch_().empty_like(u)
    out[1:-1] = (u[2:] - u[:-2]) / (2.0 * h)
    out[0] = (u[1] - u[0]) / h
    out[-1] = (u[-1] - u[-2]) / h
    return out


def torch_():
    return nat._torch()


def grad_long(rs, h: Optional[float] = None):
    """Discrete gradient of the long part, one tensor per component
    (``observables.py:142-172``): the differentiated mode's factor gets the 1D
    finite difference; Tucker factors are re-orthogonalised by a QR whose R is
    folded into the core.  Runs on the device (cuSOLVER QR)."""
    from .formats import to_device
    torch = torch_()
    if isinstance(rs, (RSCanonical, RSTucker)):
        h = rs.grid.h
        long = rs.long
    else:
        long = rs
        if h is None:
            raise ConfigError("grad_long needs the mesh size for a bare tensor")
    comps = []
    if isinstance(long, CanonicalTensor):
        facs = [to_device(f) for f in long.factors]
        w = to_device(long.weights)
        for mode in range(3):
            f = list(facs)
            f[mode] = _fd_rows(facs[mode], h)
            comps.append(CanonicalTensor(w, tuple(f)))
    elif isinstance(long, TuckerTensor):
        for mode in range(3):
            f = list(long.factors)
            q, r = torch.linalg.qr(_fd_rows(f[mode], h))
            core = torch.movedim(torch.tensordot(r, torch.movedim(long.core, mode, 0), dims=1),
                                 0, mode).contiguous()
            f[mode] = q.contiguous()
            comps.append(TuckerTensor(core, tuple(f)))
    else:
        raise ConfigError(f"grad_long cannot handle {type(long).__name__}")
    return tuple(comps)


def _pair_sums(system, reference, r_l: int, targets, mode: int):
    torch = nat._torch()
    idx, z = _system_arrays(system)
    table = to_device(reference.table)
    w = to_device(reference.tensor.weights[: r_l + 1])
    tgt = to_device(np.asarray(targets, dtype=np.int64), torch.int64)
    m = int(tgt.shape[0])
    base = torch.empty(max(m, 1), dtype=torch.float64, device="cuda")
    dsh = torch.empty((max(m, 1), 3), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().rs_pair_sums(table.data_ptr(), table.shape[1], reference.origin_index,
                                     w.data_ptr(), r_l + 1, reference.grid.h ** 3, idx.data_ptr(),
                                     z.data_ptr(), int(idx.shape[0]), tgt.data_ptr(), m, mode,
                                     base.data_ptr(), dsh.data_ptr(), nat.stream_ptr()),
              "rs_pair_sums")
    return base[:m], dsh[:m], z


def reference_energy(system, reference, split_index: Optional[int] = None) -> float:
    """Energy from windowed reference terms on the unreduced long part,
    O(N^2 R_l) (``observables.py:190-213``)."""
    r_l = reference.split_index if split_index is None else int(split_index)
    if r_l is None:
        raise ConfigError("reference carries no split index")
    count = system.count
    plong, _, z = _pair_sums(system, reference, r_l, np.arange(count), 0)
    terms = z * (plong - z * reference.self_value(r_l))
    return 0.5 * float(dd_sum(terms))


def forces_fd(system, reference, split_index: Optional[int] = None, targets=None,
              device: bool = False):
    """One-sided FD forces of the long-range energy for many particles at once
    (``force_fd`` for every target in one launch)."""
    r_l = reference.split_index if split_index is None else int(split_index)
    if r_l is None:
        raise ConfigError("reference carries no split index")
    count = system.count
    tg = np.arange(count) if targets is None else np.asarray(targets, dtype=np.int64)
    if tg.size and (tg.min() < 0 or tg.max() >= count):
        raise DomainError("particle index out of range")
    _, dsh, z = _pair_sums(system, reference, r_l, tg, 1)
    torch = nat._torch()
    zt = z[to_device(tg, torch.int64)]
    f = (zt[:, None] * dsh) / system.grid.h
    return f if device else to_host(f)


def forces_fd_scale(system, reference, split_index: Optional[int] = None, targets=None,
                    device: bool = False):
    """Cancellation scale of :func:`forces_fd`, per target and axis:
    ``|z_j| sum_{p != j} |z_p| (|pl(o - e_a)| + |pl(o)|) / h`` -- the magnitude
    the one-sided difference ``observables.py:253-256`` cancels from.  Two
    correctly rounded evaluations of the force (the reference's ``math.fsum``
    and the double-double sum here) agree to a few ulp of THIS number, not of
    the force itself; the parity tests state their tolerance against it."""
    r_l = reference.split_index if split_index is None else int(split_index)
    if r_l is None:
        raise ConfigError("reference carries no split index")
    count = system.count
    tg = np.arange(count) if targets is None else np.asarray(targets, dtype=np.int64)
    if tg.size and (tg.min() < 0 or tg.max() >= count):
        raise DomainError("particle index out of range")
    _, dsh, z = _pair_sums(system, reference, r_l, tg, 2)
    torch = nat._torch()
    zt = z[to_device(tg, torch.int64)].abs()
    f = (zt[:, None] * dsh) / system.grid.h
    return f if device else to_host(f)


def force_fd(system, j: int, reference, split_index: Optional[int] = None,
             support_radius: Optional[float] = None) -> ForceVector:
    """Force on particle ``j`` (``observables.py:216-259``)."""
    r_l = reference.split_index if split_index is None else int(split_index)
    if r_l is None:
        raise ConfigError("reference carries no split index")
    if not (0 <= j < system.count):
        raise DomainError(f"particle index {j} out of range")
    if support_radius is not None:
        h = system.grid.h
        pos = to_host(system.base.positions)
        idx = to_host(system.indices)
        others = np.arange(system.count) != j
        for axis in range(3):
            moved = system.grid.position(idx[j]) - np.eye(3)[axis] * h
            dist = np.linalg.norm(pos[others] - moved, axis=1)
            if float(dist.min(initial=np.inf)) < support_radius:
                raise SeparationError(f"shifting particle {j} along axis {axis} enters another "
                                      "particle's short-range window")
    f = forces_fd(system, reference, r_l, targets=[j])
    return ForceVector(index=j, force=f[0])


# ----------------------------------------------------------- direct oracles
def direct_energy(system: ParticleSystem) -> float:
    """Exact Newton pair sum (validation helper, ``observables.py:77-86``)."""
    if system.count < 2:
        return 0.0
    pos, q = system.positions, system.charges
    terms = []
    for i in range(system.count - 1):
        d = np.sqrt(np.sum((pos[i + 1:] - pos[i]) ** 2, axis=1))
        if d.size and d.min() <= 0.0:
            raise SingularityError("coincident particles make the energy singular")
        terms.append(q[i] * q[i + 1:] / d)
    return math.fsum(np.concatenate(terms))


def direct_force(system: ParticleSystem, j: int) -> ForceVector:
    """Exact Newton force ``z_j sum z_k (x_j - x_k)/r^3`` (``observables.py:262-274``)."""
    if not (0 <= j < system.count):
        raise DomainError(f"particle index {j} out of range")
    diff = system.positions[j] - system.positions
    r2 = np.sum(diff * diff, axis=1)
    r2[j] = 1.0
    if np.any(r2[np.arange(system.count) != j] <= 0.0):
        raise SingularityError("coincident particles make the force singular")
    scale = system.charges[j] * system.charges / np.power(r2, 1.5)
    scale[j] = 0.0
    return ForceVector(index=j, force=np.asarray([math.fsum(scale * diff[:, a]) for a in range(3)]))
