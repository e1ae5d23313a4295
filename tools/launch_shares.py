"""Launch list (ncu --metrics gpu__time_duration.sum --csv) -> share of device
time per kernel, excluding the bench's DGEMM/L2 peak probes and L2 flush."""
import csv
import io
import sys
from collections import defaultdict

path = sys.argv[1]
txt = open(path).read()
txt = txt[txt.index('"ID"'):]
tot, cnt = defaultdict(float), defaultdict(int)
for r in csv.DictReader(io.StringIO(txt)):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")[:70]
    # our kernels (rsb::, the anonymous-namespace k_* ones, the CUB node sort);
    # torch's L2-flush fill and the DGEMM/L2 peak probes are not part of the step
    if not (name.startswith("rsb::") or "::k_" in name or name.startswith("k_")
            or name.startswith("cub::")) or "l2_probe" in name:
        continue
    v = float(r["Metric Value"])
    unit = r["Metric Unit"]
    v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
    tot[name] += v
    cnt[name] += 1
S = sum(tot.values())
print("| kernel | launches | total us | share |")
print("|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / S:.3f} |")
print(f"\nTotal: {S:.1f} us over the listed launches.")
