"""Multi-rank host logic of the sharded path, world_size 2 on CPU (gloo)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_09218_b200 import configs
from paper_1606_09218_b200.parallel import (particle_shard, plane_costs, shift_histogram_host,
                                             sharded_sum, slab_bounds)
import paper_1606_09218_b200 as rt


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, idx, z, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = particle_shard(idx.shape[0], rank, world)
    part = torch.from_numpy(shift_histogram_host(idx[lo:hi], z[lo:hi], n))
    sharded_sum(part, dist.group.WORLD)
    q.put((rank, part.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_histogram_allreduce_gloo():
    s = configs.system("C2")
    grid = rt.Grid3(256, rt.Box3(16.0))
    idx = rt.snap_to_grid(s, grid).indices
    z = np.asarray(s.charges)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, idx, z, 256, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = shift_histogram_host(idx, z, 256)
    assert np.array_equal(out[0], out[1])          # every rank gets identical bytes
    assert np.allclose(out[0], full, rtol=1e-14, atol=0)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_particle_shards_partition(world):
    for count in (1, 7, 1000, 100003):
        if count < world:
            continue
        ranges = [particle_shard(count, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == count
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        sizes = [b - a for a, b in ranges]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_slab_bounds_balanced(world):
    s = configs.system("C3")
    grid = rt.Grid3(512, rt.Box3(40.0))
    idx = rt.snap_to_grid(s, grid).indices
    costs = plane_costs(idx, 92, 512)
    # plane cost = n^2 + exact pair count per plane
    lo = np.maximum(idx - 92, 0)
    hi = np.minimum(idx + 92, 511)
    pairs = np.prod(hi - lo + 1, axis=1).sum()
    assert np.isclose(costs.sum(), 512 ** 3 + pairs)
    b = slab_bounds(costs, world)
    assert b[0] == 0 and b[-1] == 512 and all(x < y for x, y in zip(b, b[1:]))
    shares = [costs[x:y].sum() / costs.sum() for x, y in zip(b, b[1:])]
    assert max(shares) <= 1.0 / world + 0.01
