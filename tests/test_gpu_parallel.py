"""The sharded (multi-rank) path of build_rs + dense_rs, executed: world size 2
on ONE GPU, gloo backend on CUDA tensors (the box has a single GPU; NCCL
refuses two ranks per device).  The ranks never wait on each other's kernels:
each collective is a host-staged gloo call on its own stream-ordered data.

Per rank: shift histograms of its particle shard -> all_reduce; the eigen
block of its modes (l mod world) -> broadcast; the bucket-K (or particle-K)
core partial of its x3 buckets / particles -> all_reduce; its work-balanced
x1 slab of the grid (no collective on the data path).  Checked: both ranks
hold bitwise the same ranks, factors and core; the slabs tile the 1-rank grid
to 1e-11 of its max (the core's K sum is split differently, so not bitwise;
measured 1e-12 at C4).
"""
import os
import socket

import numpy as np
import pytest

from paper_1606_09218_b200 import configs

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    import paper_1606_09218_b200 as rt
    from oracle import rs_oracle as orc
    if name.startswith("tiny"):
        c = orc.small_case(n=32, count=24, seed=5, kind="yukawa")
        cfg = rt.AssemblyConfig(grid=rt.Grid3(32, rt.Box3(8.0)),
                                kernel=rt.RadialKernel("yukawa", c["lam"]), M=15, split_index=7,
                                sigma=1.0, delta=1e-6, long_format="tucker",
                                reduction=rt.ReductionConfig(eps=1e-8, max_sweeps=0),
                                max_overlap=None)
        return rt.ParticleSystem(c["positions"], c["charges"], rt.Box3(8.0)), cfg
    return configs.system(name), configs.assembly_config(name)


def _worker(rank, world, port, name, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_1606_09218_b200 as rt
    from paper_1606_09218_b200.parallel import plane_costs, slab_bounds
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    system, cfg = _case(name)
    n = cfg.grid.n
    plan = rt.plan_for(cfg, cfg.split_index)
    idx = rt.snap_to_grid(system, cfg.grid).indices
    b = slab_bounds(plane_costs(idx, plan.gamma, n), world)
    lo, hi = b[rank], b[rank + 1]
    res = rt.build_rs(system, cfg, group=dist.group.WORLD, prefetch_dense=(lo, hi))
    slab = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(lo, hi))
    # a few planes + checksums instead of the whole slab (C4: 4 GB per rank)
    planes = sorted({lo, (lo + hi) // 2, hi - 1})
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             ranks=np.array(res.report["tucker_ranks"]), lo=lo, hi=hi,
             core=res.rs.long.core.cpu().numpy(),
             f0=res.rs.long.factors[0].cpu().numpy(), f2=res.rs.long.factors[2].cpu().numpy(),
             plane_sums=slab.sum(dim=(1, 2)).cpu().numpy(),
             plane_abs=slab.abs().amax(dim=(1, 2)).cpu().numpy(),
             planes=np.array(planes),
             plane_vals=np.stack([slab[p - lo].cpu().numpy() for p in planes]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["tiny_eigh", "C2", "C4"])
def test_two_rank_build_and_slabs(cuda, tmp_path, name):
    import torch
    import torch.multiprocessing as mp
    import paper_1606_09218_b200 as rt
    if name == "C4" and torch.cuda.get_device_properties(0).total_memory < 60 << 30:
        pytest.skip("C4 needs a large device")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
        assert p.exitcode == 0
    out = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(2)]
    # identical decisions and factors on both ranks
    assert np.array_equal(out[0]["ranks"], out[1]["ranks"])
    for key in ("core", "f0", "f2"):
        assert np.array_equal(out[0][key], out[1][key]), key
    assert out[0]["lo"] == 0 and out[0]["hi"] == out[1]["lo"] and out[1]["hi"] == _case(name)[1].grid.n
    # against the single-rank result
    system, cfg = _case(name)
    res = rt.build_rs(system, cfg)
    assert list(out[0]["ranks"]) == res.report["tucker_ranks"]
    core1 = res.rs.long.core.cpu().numpy()
    assert np.max(np.abs(out[0]["core"] - core1)) <= 1e-12 * np.max(np.abs(core1))
    g = rt.dense_rs(res.rs, limit=1 << 62, device=True)
    scale = float(g.abs().max())
    sums = g.sum(dim=(1, 2)).cpu().numpy()
    n = cfg.grid.n
    for o in out:
        lo, hi = int(o["lo"]), int(o["hi"])
        assert np.max(np.abs(o["plane_sums"] - sums[lo:hi])) <= 1e-12 * scale * n * n
        for p, v in zip(o["planes"], o["plane_vals"]):
            assert np.max(np.abs(v - g[int(p)].cpu().numpy())) <= 1e-11 * scale, (name, p)
