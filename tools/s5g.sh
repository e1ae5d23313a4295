#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "kernels or reference_large or large or parity or prefetch" > $O/s5g_pytest.txt 2>&1
tail -4 $O/s5g_pytest.txt
python bench.py --no-cpu-baseline > $O/s5g_bench_C5.json 2> $O/s5g_bench_C5.err
RSB200_TUCKER_OZ=0 python bench.py --no-cpu-baseline > $O/s5g_bench_C5_dmma.json 2> $O/s5g_bench_C5_dmma.err
python - <<'P'
import json
for f in ("s5g_bench_C5", "s5g_bench_C5_dmma"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["stages_ms_per_step"].items() if v}, d["clocks"]["reasons"], d["roofline"]["kernel"][:30], d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
P
tail -3 $O/s5g_bench_C5.err
