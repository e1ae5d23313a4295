"""Copy a profiling pass (tools/profile_round2.sh, TAG) from gpurun_out/ into
profiles/: bench lines, launch shares + list, ncu summaries (one file), raw
metric pages (gzipped) and the per-kernel DRAM traffic table bench.py reads
for `roofline.traffic` (profiles/<TAG>_ncu_traffic.json)."""
import glob, gzip, json, os, re, shutil, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = "gpurun_out", "profiles"
units = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}


def val(s):
    m = re.match(r"([-\d\.nan]+) (\w+)", s)
    if not m or "nan" in m.group(1):
        return None
    return float(m.group(1)) * units.get(m.group(2), 1)


def key_of(name):
    for k, v in (("k_short_mma", "short_mma"), ("k_tucker_gemm_res", "tucker_gemm_res"), ("k_oz_res", "oz_res"),
                 ("k_tucker_apply", "tucker_apply"), ("syrk", "syrk"), ("core_h", "core_h")):
        if k in name:
            return v
    return name


out = {}
for c in ("C2", "C3", "C4", "C5"):
    path = f"{G}/{tag}_ncu_summary_{c}.md"
    if not os.path.exists(path):
        continue
    out[c] = {}
    for line in open(path).read().splitlines():
        if not line.startswith("|") or "kernel" in line or "---" in line:
            continue
        f = [x.strip() for x in line.strip("|").split("|")]
        rd, wr = val(f[2]), val(f[3])
        out[c][key_of(f[0])] = {
            "dram_bytes_per_launch": (rd + wr) if rd is not None and wr is not None else None,
            "dram_read": rd, "dram_write": wr, "duration": f[1], "dmma_pipe_pct": f[10]}
json.dump(out, open(f"{P}/{tag}_ncu_traffic.json", "w"), indent=1)
with open(f"{P}/{tag}_ncu_summary.md", "w") as fh:
    fh.write(f"# Round 2 ({tag}) -- ncu --set full summaries\n\n`tools/profile_round2.sh` (TAG={tag}; "
             "ordinary streams (RSB200_SIDE_SMS=0: ncu cannot replay on the green-context side "
             "stream), one launch per kernel after the warm-up steps of `bench.py --config Cx "
             "--steps 1 --warmup 3`); tables by `tools/ncu_summary.py`, raw metric pages in "
             f"`{tag}_ncu_raw_Cx.csv.gz`.  `dmma_*%` = `sm__inst_executed_pipe_tensor_subpipe_dmma` / "
             "`sm__pipe_tensor_subpipe_dmma_cycles_active` (% of peak sustained active): FP64 "
             "tensor math is DMMA, which the `fp64` pipe counters do not see.  `-nan` rows: "
             "launches ncu could not replay inside the chained call (the other configs' rows "
             "carry that kernel's counters).\n")
    for c in ("C5", "C4", "C3", "C2"):
        path = f"{G}/{tag}_ncu_summary_{c}.md"
        if os.path.exists(path):
            fh.write(open(path).read().replace(f"{G}/{tag}_full_", f"{tag}_full_"))
for f in glob.glob(f"{G}/{tag}_bench_*.json") + [f"{G}/{tag}_launch_shares_C5.md",
                                                  f"{G}/{tag}_launches_C5.csv.gz", f"{G}/{tag}_smi.txt",
                                                  f"{G}/{tag}_sass_counts.txt",
                                                  f"{G}/{tag}_pytest_gpu.txt"]:
    if os.path.exists(f):
        shutil.copy(f, f"{P}/" + os.path.basename(f))
for c in ("C2", "C3", "C4", "C5"):
    src = f"{G}/{tag}_ncu_raw_{c}.csv"
    if os.path.exists(src):
        with open(src, "rb") as a, gzip.open(f"{P}/{tag}_ncu_raw_{c}.csv.gz", "wb") as b:
            b.write(a.read())
print("collected", tag, {c: list(v) for c, v in out.items()})
