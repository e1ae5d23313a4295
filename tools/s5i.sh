#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "reference_large or large or parallel" > $O/s5i_pytest.txt 2>&1
tail -3 $O/s5i_pytest.txt
for c in C5 C4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/s5i_bench_$c.json 2> $O/s5i_bench_$c.err
  RSB200_CORE_H=cuda timeout 600 python bench.py --config $c --no-cpu-baseline > $O/s5i_bench_${c}_cuda.json 2> $O/s5i_bench_${c}_cuda.err
done
for f in $O/s5i_bench_C*.json; do python - "$f" <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"], 3), {k: round(v, 2) for k, v in d["stages_ms_per_step"].items() if v}, d["clocks"]["reasons"])
P
done
