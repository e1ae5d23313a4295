#!/bin/bash
# Bench lines + GPU suite at the final binary (TAG files replace the earlier pass's)
TAG=${TAG:-r02}
O=gpurun_out
python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.txt 2>&1
tail -2 $O/${TAG}_pytest_gpu.txt
python bench.py > $O/${TAG}_bench_C5.json 2> $O/${TAG}_bench_C5.err
RSB200_TUCKER_OZ=0 python bench.py --no-cpu-baseline > $O/${TAG}_bench_C5_dmma_tucker.json 2> $O/${TAG}_bench_C5_dmma_tucker.err
for c in C4 C3 C2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference_C5.json 2> $O/${TAG}_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.txt 2>&1; tail -2 $O/${TAG}_smoke.txt
for f in $O/${TAG}_bench_C*.json; do python - "$f" <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"], 3), d["clocks"]["reasons"])
P
done
