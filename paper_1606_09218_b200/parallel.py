"""Multi-GPU decomposition of the RS path (one process per GPU, torchrun).

Two axes shard naturally:

* grid assembly along x1: contiguous slabs ``[lo, hi)`` whose boundaries
  balance the per-plane work (pairs of (plane point, covering copy) plus the
  n^2 store), so each rank writes only its slab -- no collective on the data
  path;
* the long-range reduction along particles: shift histograms and RHOSVD core
  partials of a particle shard, summed with one ``all_reduce`` each (NCCL over
  NVLink on the GPU box, gloo in the CPU tests).  The eigen-truncation then
  runs replicated on bitwise-identical Grams (all_reduce delivers the same
  bytes to every rank), so all ranks agree on ranks and factors.
"""

from __future__ import annotations

import numpy as np


def plane_costs(indices: np.ndarray, gamma: int, n: int) -> np.ndarray:
    """Work per x1 plane: n^2 stores + sum over copies covering the plane of
    their clipped (x2, x3) window area."""
    cost = np.full(n, float(n) * n)
    if gamma <= 0 or indices.shape[0] == 0:
        return cost
    lo = np.maximum(indices - gamma, 0)
    hi = np.minimum(indices + gamma, n - 1)
    area = ((hi[:, 1] - lo[:, 1] + 1) * (hi[:, 2] - lo[:, 2] + 1)).astype(np.float64)
    diff = np.zeros(n + 1)
    np.add.at(diff, lo[:, 0], area)
    np.add.at(diff, hi[:, 0] + 1, -area)
    return cost + np.cumsum(diff[:n])


def slab_bounds(costs: np.ndarray, world: int) -> list:
    """Contiguous boundaries ``b_0 = 0 < ... < b_world = n`` with near-equal
    prefix cost per slab (every slab non-empty when n >= world)."""
    n = int(costs.shape[0])
    if world <= 1:
        return [0, n]
    c = np.concatenate([[0.0], np.cumsum(costs)])
    total = c[-1]
    bounds = [0]
    for r in range(1, world):
        b = int(np.searchsorted(c, total * r / world))
        b = max(b, bounds[-1] + 1)
        b = min(b, n - (world - r))
        bounds.append(b)
    bounds.append(n)
    return bounds


def particle_shard(count: int, rank: int, world: int) -> tuple:
    """Contiguous particle range of ``rank`` (remainder spread over low ranks)."""
    base, rem = divmod(count, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def sharded_sum(tensor, group=None):
    """In-place sum over the ranks of ``group`` (no-op without a process group)."""
    import torch.distributed as dist

    if group is None or not dist.is_available() or not dist.is_initialized():
        return tensor
    if dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def shift_histogram_host(indices: np.ndarray, charges: np.ndarray, n: int) -> np.ndarray:
    """Host statement of ``rs_shift_hist`` (3, n): c[l, s] = sum z^2 over the
    copies whose mode-l window starts at s = n - j_l.  Used by the CPU tests of
    the sharded path."""
    c = np.zeros((3, n))
    for l in range(3):
        np.add.at(c[l], n - indices[:, l], charges * charges)
    return c
