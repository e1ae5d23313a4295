O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_large.py tests/test_gpu_next.py -x -q -k "not C3" > $O/r02s_pytest.log 2>&1
tail -2 $O/r02s_pytest.log | cut -c1-200
for c in C5 C4; do
  BENCH_NO_OBSERVABLES=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 2>$O/r02s_$c.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step'],2), {k:round(v,1) for k,v in d['stages_ms_per_step'].items() if v})"
done
