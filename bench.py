#!/usr/bin/env python
"""RS potential-sum assembly benchmark (driver contract: one JSON line on rank 0).

Workload (default ``--config C2`` = BASELINE.json configs[1]): Newton kernel,
N = 1000 particles on a jittered 10^3 lattice, n = 256, R = 28 (R_l = R_s = 14),
eps = 1e-6, delta = 1e-8.  One *step* = one full RS assembly of the particle
system into the dense fp64 grid through the package API:
``build_rs`` (snap, shift-merged Gram on DMMA, eigh, rank selection, RHOSVD
core) + ``assemble_grid`` (fused Tucker + short-range plane GEMM).  The host
prologue (quadrature calibration, (2n,R) table: depends only on the grid
configuration) is planned once before timing, like an FFT plan.

* ``value``  -- grid points per second, inputs resident in HBM, device time
  (CUDA events), L2 flushed (256 MiB write) before every timed step.
* ``e2e``    -- same metric through the public API from pinned HOST buffers:
  H2D of positions/charges + assembly + D2H of the whole grid, every step.
* ``roofline`` -- the dominant kernel (plane GEMM, ``gemm_plane``) timed live
  with CUDA events around its launches; algorithmic flops per SURVEY 8(d):
  2 P (short-range pairs) + 2 r3 n^3 (last Tucker mode); peak = a cuBLAS
  DGEMM 8192^3 measured live in this process (MEASURED_PEAKS.json has no FP64).
* ``cpu_baseline`` -- the reference algorithm (oracle port, numpy + OpenBLAS
  on all host cores; the reference's dense_cct loop is single-threaded) on
  the same workload, dense_cct on a deterministic particle subsample and
  extrapolated by exact pair counts.

``--impl reference`` runs only that CPU path (rank 0; other ranks exit 0).
Multi-GPU (torchrun): each rank assembles a work-balanced x1 slab of the same
grid (strong scaling); build_rs is replicated (deterministic, bitwise equal).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=8.0,
                    help="reference arm: measured CPU seconds per sampled step")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def workload_desc(name):
    from paper_1606_09218_b200 import configs
    m = configs.MANIFEST[name]
    return {"workload": f"{name}: {m['kernel']} kernel, N={m['N']}, n={m['n']}, b={m['b']}, "
                        f"R={m['M'] + 1} (R_l={m['split_index'] + 1}, "
                        f"R_s={m['M'] - m['split_index']}), eps={m['eps']}, delta={configs.DELTA}",
            "N": m["N"], "n": m["n"], "kernel": m["kernel"],
            "step": "build_rs + dense grid assembly (plan = host quadrature/table, built once)"}


def pair_counts(idx, gamma, n):
    lo = np.maximum(idx - gamma, 0)
    hi = np.minimum(idx + gamma, n - 1)
    return np.prod(hi - lo + 1, axis=1).astype(np.float64)


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    In-process NVML queries (three cheap calls per sample, every 5 ms) from a
    background thread; nvidia-smi polling was measured to stall this
    host-latency-sensitive step by ~0.6 ms per sample.  Falls back to
    nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.stop = threading.Event()
        self.thread = None
        self.nvml = None
        self.period = float(os.environ.get("BENCH_CLOCK_MS", "10")) / 1e3

    def _sample(self, h):
        nv = self.nvml
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.rows.append((sm, mx, rs))
        except Exception:
            pass

    def _run(self, h):
        # first sample one period in: the NVML calls contend with the CUDA
        # driver calls of the step being launched
        while not self.stop.wait(self.period):
            self._sample(h)

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() \
                else self.device
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = nv
            self.handle = h
            self.thread = threading.Thread(target=self._run, args=(h,), daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
        return self

    def __exit__(self, *exc):
        # (called right after the timed region's closing synchronize)
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
            if not self.rows:  # region shorter than one period: one sample at its end
                self._sample(self.handle)

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"],
                    "samples": 0}
        reasons = sorted({k for _, _, r in rows for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median([r[0] for r in rows])),
                "sm_max_mhz": float(max(r[1] for r in rows)), "reasons": reasons,
                "samples": len(rows), "source": "nvml"}


# ---------------------------------------------------- CPU reference (oracle)
# Tucker ranks of the configs (the reference's own at C1-C3 and C5,
# tests/golden/{golden,large}.json; the pinned oracle's at C4): the sampled
# reference step below forces them so every stage runs at its true size.
REF_RANKS = {"C1": (8, 8, 8), "C2": (12, 12, 12), "C3": (23, 23, 23), "C4": (40, 40, 40),
             "C5": (132, 132, 132)}
_REF_CACHE: dict = {}


def reference_assembly_time(name, budget_s=8.0):
    """One step of the reference algorithm (oracle port of rstensor's
    build_rs + dense_rs: numpy / OpenBLAS on all host cores, the dense_cct
    loop single-threaded like the reference) on a BOUNDED sample of the
    workload, extrapolated stage by stage by the stage's exact cost driver:

    * snap and the three n x n eigh: full size, not scaled;
    * side matrices + A A^T Gram + projections + core: on every k-th
      particle (cost linear in the K = N R_l columns), x N / N_sample;
    * Tucker dense: on p x1 planes (linear in planes), x n / p;
    * dense_cct: on every m-th particle, x (all pairs) / (sampled pairs).

    ``budget_s`` sizes the samples (about that much measured CPU time per
    step).  Returns (extrapolated seconds, measured seconds, details)."""
    from oracle import rs_oracle as orc
    from paper_1606_09218_b200 import configs

    ent = _REF_CACHE.get(name)
    if ent is None:
        case = configs.oracle_case(name)
        p = orc.prologue(case["kind"], case["lam"], case["b"], case["n"], case["M"],
                         case["split_index"], case["delta"])  # plan (not timed: an FFT-style plan)
        ul, wl = orc.local_window(p["table"], p["w"], case["split_index"], p["gamma"])
        ent = _REF_CACHE[name] = (case, p, orc.local_dense(ul, wl))
    case, p, L0 = ent
    n, N = case["n"], case["positions"].shape[0]
    nt = case["split_index"] + 1
    ranks = REF_RANKS[name]
    z = case["charges"]
    t_all0 = time.perf_counter()
    t0 = time.perf_counter()
    idx, _, _ = orc.snap(case["positions"], case["b"], n)
    t_snap = time.perf_counter() - t0
    pc = pair_counts(idx, p["gamma"], n)
    # K-linear part: aim at ~0.35 budget (2 n^2 K flops per mode at ~3e11 flop/s)
    k_cols = max(64 * nt, int(0.35 * budget_s * 3e11 / (6.0 * n * n)))
    gstride = max(1, -(-N * nt // k_cols))
    sub = np.arange(0, N, gstride)
    t0 = time.perf_counter()
    weights, facs = orc.long_side_matrices(p["table"], p["w"], idx[sub], z[sub], case["split_index"])
    grams = [(u * np.abs(weights)) @ (u * np.abs(weights)).T for u in facs]
    t_gram = time.perf_counter() - t0
    t0 = time.perf_counter()
    zs = []
    for G in grams:
        vals, vecs = np.linalg.eigh(G)
        zs.append(vecs[:, np.argsort(vals)[::-1]])
    t_eigh = time.perf_counter() - t0
    zs = [zz[:, :r] for zz, r in zip(zs, ranks)]
    t0 = time.perf_counter()
    pr = [zz.T @ u for zz, u in zip(zs, facs)]
    t_proj = time.perf_counter() - t0
    # the core contraction (einsum, 2 r1 r2 r3 flops per column at ~3.5e9 flop/s)
    # on its own, smaller column sample: ~0.15 budget
    kc = int(max(4 * nt, min(weights.size, 0.15 * budget_s * 3.5e9 /
                             (2.0 * ranks[0] * ranks[1] * ranks[2]))))
    t0 = time.perf_counter()
    core = np.zeros(ranks)
    for lo in range(0, kc, 2048):
        hi = min(lo + 2048, kc)
        core += np.einsum("k,ak,bk,ck->abc", weights[lo:hi], pr[0][:, lo:hi], pr[1][:, lo:hi],
                          pr[2][:, lo:hi], optimize=True)
    t_core = t_proj + (time.perf_counter() - t0) * weights.size / kc   # scaled to the Gram sample
    del facs, grams, pr
    # Tucker dense on a slab of planes (2 r1 n^3-dominated: ~0.15 budget)
    planes = int(max(1, min(n, 0.15 * budget_s * 5e10 / (2.0 * ranks[0] * n * n + 1))))
    t0 = time.perf_counter()
    orc.tucker_dense(core, zs, x1=slice(0, planes))
    t_tucker = time.perf_counter() - t0
    # dense_cct on every m-th particle (~0.4 budget at ~2.3e8 pairs/s)
    want_pairs = 0.4 * budget_s * 2.3e8
    cstride = max(1, int(pc.sum() / want_pairs))
    csub = np.arange(0, N, cstride)
    t0 = time.perf_counter()
    orc.dense_cct_numpy(L0, p["gamma"], idx[csub], z[csub], n)
    t_cct = time.perf_counter() - t0
    measured = time.perf_counter() - t_all0
    frac = float(pc[csub].sum() / pc.sum())
    kscale = N / sub.size
    total = (t_snap + t_eigh + (t_gram + t_core) * kscale + t_tucker * n / planes
             + t_cct / frac)
    det = dict(measured_s=measured, extrapolated_s=total, gram_particles=int(sub.size),
               core_columns=kc,
               tucker_planes=planes, cct_stride=cstride, pair_fraction=frac,
               stages_s=dict(snap=t_snap, eigh=t_eigh, gram_x=t_gram * kscale,
                             core_x=t_core * kscale, tucker_x=t_tucker * n / planes,
                             dense_cct_x=t_cct / frac))
    return total, measured, det


def reference_sample_text(name, det, cores):
    st = det["stages_s"]
    return (f"{name} reference pipeline (oracle numpy port of rstensor build_rs + dense_rs; BLAS "
            f"on {cores} threads, dense_cct single-threaded like the reference), EXTRAPOLATED "
            f"per stage from a bounded sample: {det['measured_s']:.1f} s measured -> "
            f"{det['extrapolated_s']:.1f} s per assembly. Snap + 3 eigh at full size; Gram + "
            f"projections on {det['gram_particles']} particles (x N/sample), the core einsum on "
            f"{det['core_columns']} of their columns (x columns/sample); Tucker dense on "
            f"{det['tucker_planes']} planes (x n/planes); dense_cct on every "
            f"{det['cct_stride']}-th particle = {det['pair_fraction']:.4f} of the pairs (x 1/that). "
            f"Extrapolated stage seconds: " + ", ".join(f"{k} {v:.2f}" for k, v in st.items()))


def _ncu_traffic(name, kernel="gemm_short"):
    """dram read+write bytes per launch of the dominant kernel from the
    committed ncu --set full summary (profiles/), or None."""
    for tag in ("r02", "r01"):   # the latest committed pass that holds this kernel
        try:
            with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_traffic.json")) as fh:
                v = json.load(fh)[name][kernel]["dram_bytes_per_launch"]
            if v is not None:
                return v
        except (OSError, KeyError, ValueError):
            continue
    return None


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def run_reference(args, rank):
    """The reference arm: rank 0 alone times the reference algorithm on the
    host cores (other ranks exit 0 without work)."""
    if rank != 0:
        return
    name = args.config
    from paper_1606_09218_b200 import configs
    m = configs.MANIFEST[name]
    times, meas = [], []
    for i in range(args.warmup + args.steps):
        t, tm, det = reference_assembly_time(name, args.ref_budget)
        if i >= args.warmup:
            times.append(t)
            meas.append(tm)
    t = float(np.mean(times))
    value = m["n"] ** 3 / t
    cores = threads_used()
    line = {"impl": "reference", "metric": "rs_assembly_grid_pts_per_s", "value": value,
            "unit": "grid-pts/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded recipe, paper_1606_09218_b200/configs.py)",
            "config": workload_desc(name),
            "measured_ms_per_step": float(np.mean(meas)) * 1e3,
            "extrapolated": True,
            "cpu_baseline": {"value": value, "unit": "grid-pts/s", "cores": cores,
                             "kind": "port", "sample": reference_sample_text(name, det, cores)},
            "e2e": {"value": value, "unit": "grid-pts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm
def _hbm_peak():
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written), else the
    profiling guide's fallback."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy test)"
    except (OSError, KeyError, ValueError):
        return 6539.0, "fallback 6539 GB/s (B200_PROFILING.md)"


def measure_dgemm_peak(torch):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3 / 1e3
    del a, b
    torch.cuda.empty_cache()
    return 2 * n ** 3 / t / 1e12


def measure_l2_peak(torch, nat):
    """L2 read bandwidth (GB/s): rs_l2_probe streaming a 32 MiB buffer 200
    times from 1184 CTAs with L1-bypassing loads, CUDA events."""
    buf = torch.ones(4 << 20, dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    L = nat.lib()
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        nat.check(L.rs_l2_probe(buf.data_ptr(), buf.numel() * 8, 20, out.data_ptr(), st), "probe")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nat.check(L.rs_l2_probe(buf.data_ptr(), buf.numel() * 8, 200, out.data_ptr(), st), "probe")
    e1.record()
    torch.cuda.synchronize()
    return buf.numel() * 8 * 200 / (e0.elapsed_time(e1) / 1e3) / 1e9


def term_supports(ul, wl, gamma, drop=1e-18):
    """Host mirror of k_term_support (per-term x3 band of the plane GEMM)."""
    mx = np.abs(ul).max(axis=0)
    thr = drop * float(np.sum(np.abs(wl) * mx ** 3))
    out = []
    for k in range(ul.shape[1]):
        f = abs(wl[k]) * mx[k] ** 2
        g = 0
        for d in range(gamma, -1, -1):
            if f * max(abs(ul[gamma + d, k]), abs(ul[gamma - d, k])) > thr:
                g = d
                break
        out.append(g)
    return out


def spawn_ranks(args):
    """``--gpus N`` without a torchrun environment: launch N ranks through
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_1606_09218_b200 as rt
    from paper_1606_09218_b200 import _native as nat
    from paper_1606_09218_b200 import configs
    from paper_1606_09218_b200.parallel import plane_costs, slab_bounds

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    name = args.config
    m = configs.MANIFEST[name]
    n = m["n"]
    system = configs.system(name)
    cfg = configs.assembly_config(name)
    grid = rt.Grid3(n, rt.Box3(m["b"]))
    host_idx = rt.snap_to_grid(system, grid).indices

    # plan (host prologue) once, outside timing
    plan = rt.plan_for(cfg, cfg.split_index)
    gamma = plan.gamma
    # work-balanced x1 slab of this rank: per-plane pair count + n^2 store
    bounds = slab_bounds(plane_costs(host_idx, gamma, n), world)
    x1_lo, x1_hi = bounds[rank], bounds[rank + 1]

    pos_d = torch.tensor(system.positions, device="cuda")
    q_d = torch.tensor(system.charges, device="cuda")
    dp = rt.DeviceParticles(pos_d, q_d, system.box)
    out_shape = (max(x1_hi - x1_lo, 1), n, n)

    # two output slabs used in turn (a serving loop's reused result buffers)
    slabs = [torch.empty(out_shape, dtype=torch.float64, device="cuda") for _ in range(2)]

    def step(particles):
        step.i = getattr(step, "i", -1) + 1
        # public API: build_rs (short-range planes prefetched on a side stream,
        # overlapping the long-range reduction) + dense_rs of this rank's slab
        res = rt.build_rs(particles, cfg, prefetch_dense=(x1_lo, x1_hi),
                          group=dist.group.WORLD if world > 1 else None,
                          prefetch_groups=int(os.environ.get("BENCH_GROUPS", "1")),
                          prefetch_out=slabs[step.i % 2])
        g = rt.dense_rs(res.rs, limit=1 << 62, device=True, x1_range=(x1_lo, x1_hi))
        step.last = g
        return res

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # W warm-up steps; then, untimed as well, settle steps until 8 steps have
    # run (the caching allocator, the front-buffer pool and lazily loaded
    # kernels reach steady state) with the stage-event pool primed
    L = nat.lib()
    for i in range(max(args.warmup, 8)):
        L.rs_prof_enable(1 if i >= max(args.warmup, 8) - 2 else 0)
        flush.fill_(i & 0xFF)   # as in the timed loop (its kernel module loads lazily)
        res = step(dp)
    L.rs_prof_enable(0)
    torch.cuda.synchronize()
    ranks_used = res.report["tucker_ranks"]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier()
    launches0 = L.rs_launch_count()
    L.rs_prof_enable(1)
    # host hygiene of a latency-bound loop: collect garbage now, pause Python's
    # cyclic GC during the timed steps (BENCH_GC=1 keeps it running)
    import gc
    gc.collect()
    if not os.environ.get("BENCH_GC"):
        gc.disable()
    verbose = bool(os.environ.get("BENCH_VERBOSE"))
    if os.environ.get("BENCH_VERBOSE") == "3":
        torch.cuda.memory._record_memory_history(max_entries=100000)
    if verbose:
        mallocs0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        host_t, mallocs_t = [], []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if verbose:
                if os.environ.get("BENCH_VERBOSE") == "2":
                    mallocs_t.append(torch.cuda.memory_stats().get("num_device_alloc", 0))
                from paper_1606_09218_b200 import assembly as _asm
                if _asm._TRACE is not None:
                    if i == 1:
                        tr0 = list(_asm._TRACE)
                    _asm._TRACE.clear()
                    _asm._mark("step")
                host_t.append(time.perf_counter())
            flush.fill_(i & 0xFF)
            ev[i][0].record()
            step(dp)
            ev[i][1].record()
        torch.cuda.synchronize()
    L.rs_prof_enable(0)
    launches = L.rs_launch_count() - launches0
    barrier()
    t_steps = [a.elapsed_time(b) for a, b in ev]
    t_mean = float(np.mean(t_steps)) / 1e3
    if verbose:
        print("step ms:", " ".join(f"{t:.3f}" for t in t_steps), file=sys.stderr)
        print("host ms:", " ".join(f"{1e3 * (b - a):.3f}" for a, b in zip(host_t[:-1], host_t[1:])),
              file=sys.stderr)
        if "tr0" in locals():
            print("step-0 host trace:", " ".join(f"{a}->{b}:{1e6 * (tb - ta):.0f}us" for (a, ta), (b, tb)
                                                  in zip(tr0[:-1], tr0[1:])), file=sys.stderr)
        print("cudaMalloc per step:", [b - a for a, b in zip(mallocs_t[:-1], mallocs_t[1:])],
              file=sys.stderr)
        if os.environ.get("BENCH_VERBOSE") == "3":
            for tr in torch.cuda.memory._snapshot()["device_traces"]:
                for e in tr:
                    if e["action"] in ("segment_alloc", "segment_map"):
                        print(e["action"], e["size"], e.get("stream"), file=sys.stderr)
                        for f in e["frames"][:14]:
                            print("   ", f["filename"].split("/")[-1], f["line"], f["name"],
                                  file=sys.stderr)
        print("cudaMalloc calls in the timed region:",
              torch.cuda.memory_stats().get("num_device_alloc", 0) - mallocs0, file=sys.stderr)
    gemm_ms, gemm_n = nat.prof_query("gemm_short")
    l0_ms, l0_n = nat.prof_query("short_l0")
    mma_ms, mma_n = nat.prof_query("short_mma")
    prof = {k: nat.prof_query(k) for k in ("short_mma", "gemm_short", "gemm_tucker", "gemm_plane",
                                          "short_rows", "short_l0", "tucker_f", "topeig", "syrk",
                                          "oz_mma",
                                          "core", "shift_project")}
    tt = torch.tensor([t_mean], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())

    # ---- end to end through the public API from pinned host buffers
    pos_h = torch.tensor(system.positions).pin_memory()
    q_h = torch.tensor(system.charges).pin_memory()
    out_h = torch.empty(out_shape, dtype=torch.float64).pin_memory()
    pos_e = torch.empty_like(pos_d)
    q_e = torch.empty_like(q_d)

    def e2e_step():
        # public API as a host user calls it: inputs from pinned host memory,
        # build_rs, then dense_rs returning the grid on the host -- its
        # device->host transfer is pipelined with the plane assembly
        pos_e.copy_(pos_h, non_blocking=True)
        q_e.copy_(q_h, non_blocking=True)
        step.last = None
        mode = os.environ.get("BENCH_E2E", "pipelined")
        if mode == "prefetch":
            step(rt.DeviceParticles(pos_e, q_e, system.box))
            out_h.copy_(step.last, non_blocking=True)
        elif mode == "grouped":
            # short planes prefetched in 8 groups; each group's Tucker part and
            # device->host copy start as soon as its planes are final
            res = rt.build_rs(rt.DeviceParticles(pos_e, q_e, system.box), cfg,
                              prefetch_dense=(x1_lo, x1_hi), prefetch_groups=8,
                              group=dist.group.WORLD if world > 1 else None)
            rt.dense_rs(res.rs, limit=1 << 62, x1_range=(x1_lo, x1_hi), out=out_h)
        else:
            res = rt.build_rs(rt.DeviceParticles(pos_e, q_e, system.box), cfg,
                              group=dist.group.WORLD if world > 1 else None)
            rt.dense_rs(res.rs, limit=1 << 62, x1_range=(x1_lo, x1_hi), out=out_h)

    for _ in range(2):
        e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())
    gc.enable()

    if rank == 0:
        peak = measure_dgemm_peak(torch)
        P = float(pair_counts(host_idx, gamma, n).sum())
        r3 = ranks_used[2]
        alg_flops = 2.0 * P  # the short-range agglomeration the dominant kernel performs
        slab_frac = (x1_hi - x1_lo) / n
        gemm_avg_s = gemm_ms / max(gemm_n, 1) / 1e3
        launches_per_step = max(gemm_n, 1) / args.steps
        achieved = alg_flops * slab_frac / launches_per_step / gemm_avg_s / 1e12 if gemm_n else None
        # executed flops of the banded GEMM: per column tile and short term k,
        # the occupied x3 buckets within that term's support gk of the tile
        bc3 = np.unique(host_idx[:, 2])
        gk = term_supports(plan.local_ul.cpu().numpy(), plan.local_wl.cpu().numpy(), gamma)
        keff = []
        for t0 in range(0, n, 64):
            for g in gk:
                lo_x, hi_x = t0 - g, min(n - 1, t0 + 63) + g
                keff.append(np.count_nonzero((bc3 >= lo_x) & (bc3 <= hi_x)))
        exec_flops = 2.0 * n * n * 64 * float(np.sum(keff))
        if mma_n:    # short range by the fused tensor-core kernel (the default)
            mma_avg_s = mma_ms / mma_n / 1e3
            ach = alg_flops * slab_frac / (mma_n / args.steps) / mma_avg_s / 1e12
            roof = {"bound": "tensor",
                    "kernel": "k_short_mma fused short-range agglomeration on DMMA (short_mma)",
                    "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": _ncu_traffic(name, "short_mma"),
                    "peak_source": "cuBLAS DGEMM 8192^3 measured live (fp64; "
                                   "MEASURED_PEAKS.json has no FP64 entry)",
                    "algorithmic_flops_per_launch": alg_flops * slab_frac / (mma_n / args.steps),
                    "note": "algorithmic = 2 flops per (grid point, covering copy) pair "
                            "(SURVEY 8d); the separable form executes more: every (tile, "
                            "x3 bucket, live term) column is a full 128 x 64 MMA column",
                    "avg_launch_ms": mma_avg_s * 1e3}
        elif gemm_n:   # short range on the plane GEMM (FP64 tensor cores)
            roof = {"bound": "tensor",
                    "kernel": "k_gemm_plane short-range plane GEMM (gemm_short)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": (achieved / peak) if achieved else None,
                    "traffic": _ncu_traffic(name),
                    "peak_source": "cuBLAS DGEMM 8192^3 measured live (fp64; "
                                   "MEASURED_PEAKS.json has no FP64 entry)",
                    "algorithmic_flops_per_step": alg_flops,
                    "executed_flops_upper_bound_per_step": exec_flops,
                    "avg_launch_ms": gemm_avg_s * 1e3}
        else:        # low overlap: dense-L0 gather, bound by L2 reads (8 B per pair)
            l2 = measure_l2_peak(torch, nat)
            l0_avg_s = l0_ms / max(l0_n, 1) / 1e3
            alg_bytes = 8.0 * P * slab_frac / (max(l0_n, 1) / args.steps)
            ach = alg_bytes / l0_avg_s / 1e9 if l0_n else None
            roof = {"bound": "l2", "kernel": "k_short_l0 dense-L0 gather (short_l0)",
                    "achieved": ach, "peak": l2, "unit": "GB/s",
                    "frac": (ach / l2) if ach else None,
                    "traffic": _ncu_traffic(name, "short_l0"),
                    "peak_source": "rs_l2_probe: 32 MiB L2-resident buffer, L1-bypassing "
                                   "8-byte loads, measured live",
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "note": "one 8-byte L0 read per (grid point, covering copy) pair; the "
                            "grid store (8 B per point) goes to HBM",
                    "avg_launch_ms": l0_avg_s * 1e3}
        # the two other kernels the north star names: the Tucker part of the slab
        # (HBM: read + write 8 B per point when accumulating into the prefetched
        # short-range slab) and the shift Gram (FP64 tensor cores)
        hbm = _hbm_peak()
        secondary = {}
        t_ms, t_n = prof["gemm_tucker"]
        if t_n and r3 <= 32:   # k_tucker_apply: 2 r3 flops per 16 bytes moved -> HBM
            t_avg = t_ms / t_n / 1e3
            tb = 16.0 * (x1_hi - x1_lo) * n * n / (t_n / args.steps)
            secondary["tucker"] = {
                "bound": "hbm", "kernel": "k_tucker_apply Tucker part accumulated into the slab "
                                          "(gemm_tucker)",
                "achieved": tb / t_avg / 1e9, "peak": hbm[0], "unit": "GB/s",
                "frac": tb / t_avg / 1e9 / hbm[0], "peak_source": hbm[1],
                "algorithmic_bytes_per_launch": tb, "avg_launch_ms": t_avg * 1e3}
        elif t_n and prof.get("oz_mma", (0.0, 0))[1]:
            # 96 < r3 <= 160 (C5): Ozaki-split GEMM on the int8 tensor cores (tcgen05, k_oz_res).
            # Its floor is the slab update itself: 8 B read + 8 B written per grid point.
            t_avg = t_ms / t_n / 1e3
            pts = float((x1_hi - x1_lo) * n * n) / (t_n / args.steps)
            tb, tf = 16.0 * pts, 2.0 * r3 * pts
            kpad = 32 * -(-r3 // 32)
            int8_ops = 28 * 2.0 * kpad * pts      # 7 slices: 28 slice products with p + q < 7
            secondary["tucker"] = {
                "bound": "hbm", "kernel": "k_oz_res Ozaki-split Tucker GEMM on tcgen05 int8 (7 slices, "
                                          "TMEM accumulators), accumulated into the slab (gemm_tucker)",
                "achieved": tb / t_avg / 1e9, "peak": hbm[0], "unit": "GB/s",
                "frac": tb / t_avg / 1e9 / hbm[0], "peak_source": hbm[1],
                "algorithmic_bytes_per_launch": tb, "avg_launch_ms": t_avg * 1e3,
                "fp64_equivalent_tflops": tf / t_avg / 1e12,
                "fp64_equivalent_vs_dgemm_peak": tf / t_avg / 1e12 / peak,
                "int8_tops_executed": int8_ops / t_avg / 1e12,
                "note": "2 r3 flops per grid point in FP64-equivalent terms (above the FP64 DMMA "
                        "roofline because the products run as exact int8 slice MMAs); the "
                        "operands' slicing is in tucker_f"}
        elif t_n:              # large r3 (C4): the plane GEMM, FP64-bound
            t_avg = t_ms / t_n / 1e3
            tf = 2.0 * r3 * (x1_hi - x1_lo) * n * n / (t_n / args.steps)
            secondary["tucker"] = {
                "bound": "tensor", "kernel": "k_tucker_gemm_res<64, true> A-resident Tucker "
                                             "GEMM accumulated into the slab (gemm_tucker)",
                "achieved": tf / t_avg / 1e12, "peak": peak, "unit": "TFLOP/s",
                "frac": tf / t_avg / 1e12 / peak, "note": "2 r3 flops per grid point",
                "algorithmic_flops_per_launch": tf, "avg_launch_ms": t_avg * 1e3}
        s_ms, s_n = prof["syrk"]
        if s_n:
            s_avg = s_ms / s_n / 1e3
            R_l = int(plan.w_long_abs.shape[0])
            # occupied shifts per mode (n - j_l distinct values) x R_l columns
            k_occ = [len(np.unique(host_idx[:, l])) * R_l for l in range(3)]
            gf = float(n * (n + 1) * sum(k_occ)) / (s_n / args.steps)
            secondary["gram"] = {
                "bound": "tensor", "kernel": "k_syrk_part shift-Gram SYRK on DMMA (syrk)",
                "achieved": gf / s_avg / 1e12, "peak": peak, "unit": "TFLOP/s",
                "frac": gf / s_avg / 1e12 / peak,
                "note": "sum over the 3 modes of n(n+1) K_l, K_l = occupied shifts x R_l "
                        f"= {k_occ} (the reference's A A^T has K = N R_l = "
                        f"{host_idx.shape[0] * R_l} columns, equal up to merging equal shifts)",
                "algorithmic_flops_per_launch": gf, "avg_launch_ms": s_avg * 1e3}
        # the other outputs BASELINE names for this config (configs[4]: per-particle
        # potential and forces): timed once, outside the assembly's timed region
        obs = None
        if world == 1 and not os.environ.get("BENCH_NO_OBSERVABLES"):
            def timed(fn, reps=3):
                fn()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    fn()
                b.record()
                torch.cuda.synchronize()
                return a.elapsed_time(b) / reps
            sysd = res.system
            obs = {"particles": int(m["N"]),
                   "particle_potentials_ms": timed(lambda: rt.particle_potentials(
                       res.rs, sysd, res.reference, device=True)),
                   "eval_rs_many_all_nodes_ms": timed(lambda: rt.eval_rs_many(
                       res.rs, sysd.indices, device=True)),
                   "forces_fd_all_particles_ms": timed(lambda: rt.forces_fd(
                       sysd, res.reference, device=True), reps=1),
                   "reference_energy_ms": timed(lambda: rt.reference_energy(sysd, res.reference),
                                                reps=1),
                   "note": "device results, no host copy; forces_fd / reference_energy are the "
                           "O(N^2 R_l) windowed pair sums (observables.py:190-259)"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            tc, _, det = reference_assembly_time(name, 20.0)   # ~20 s of CPU work
            cpu = {"value": n ** 3 / tc, "unit": "grid-pts/s", "cores": threads_used(),
                   "kind": "port", "sample": reference_sample_text(name, det, threads_used())}
        clocks = clk.summary()
        line = {
            "metric": "rs_assembly_grid_pts_per_s",
            "value": n ** 3 / t_max,
            "unit": "grid-pts/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max * 1e3,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded recipe, paper_1606_09218_b200/configs.py)",
            "config": {**workload_desc(name), "parallelism": f"x1-slabs x{world}",
                       "l2": "flushed (256 MiB write) before each timed step",
                       "tucker_ranks": ranks_used, "gamma": gamma},
            "gbs": 8.0 * n ** 3 / t_max / 1e9,
            "clocks": clocks,
            "e2e": {"value": n ** 3 / t_e2e, "unit": "grid-pts/s",
                    "h2d_bytes_per_step": int(pos_h.numel() * 8 + q_h.numel() * 8),
                    "d2h_bytes_per_step": int(out_h.numel() * 8), "ms_per_step": t_e2e * 1e3},
            "gpu_launches": int(launches),
            "roofline": roof,
            "secondary_rooflines": secondary,
            # (oz_mma is the tcgen05 kernel inside gemm_tucker: not a stage of its own)
            "stages_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if k != "oz_mma"},
            "observables": obs,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
