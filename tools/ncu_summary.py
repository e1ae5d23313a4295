"""Summarise ncu --set full reports: per kernel launch, duration, DRAM bytes,
L2 hit rate, occupancy, DMMA / tensor pipe and top stall reasons (markdown rows)."""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "lts__t_sector_hit_rate.pct": "l2_hit",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active%",
    "launch__registers_per_thread": "regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem%",
    # FP64 tensor math on sm_100a is DMMA: it issues on the tensor pipe's dmma
    # sub-pipe, so sm__pipe_fp64_* / sm__inst_executed_pipe_fp64 read 0 for it
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst%",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe%",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active": "tensor_inst%",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe%",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64inst%",
    "lts__t_bytes.sum": "l2_bytes",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not h.endswith("_not_issued")]
    for d in data:
        rec = {"kernel": d[idx["Kernel Name"]].split("(")[0].replace("void ", "")}
        for k, v in WANT.items():
            if k in idx:
                rec[v] = d[idx[k]] + " " + units[idx[k]]
        st = sorted(((float(d[idx[h]] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for h in stall), reverse=True)[:3]
        rec["top stalls"] = ", ".join(f"{n}" for _, n in st)
        yield rec


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"\n### {rep}\n")
        recs = list(rows(rep))
        keys = list(recs[0].keys()) if recs else []
        print("| " + " | ".join(keys) + " |")
        print("|" + "---|" * len(keys))
        for r in recs:
            print("| " + " | ".join(str(r.get(k, "")) for k in keys) + " |")
