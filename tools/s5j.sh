#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "oz_gemm or tucker_gemm" > $O/s5j_pytest.txt 2>&1
tail -3 $O/s5j_pytest.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "reference_large or large" >> $O/s5j_pytest.txt 2>&1
tail -2 $O/s5j_pytest.txt
timeout 600 python bench.py --config C5 --no-cpu-baseline > $O/s5j_bench_C5.json 2> $O/s5j_bench_C5.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/s5j_bench_C5.json").read().strip().splitlines()[-1])
print(round(d["ms_per_step"], 3), {k: round(v, 2) for k, v in d["stages_ms_per_step"].items() if v}, d["clocks"]["reasons"])
P
