O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > $O/r02s_pytest.log 2>&1
tail -4 $O/r02s_pytest.log | cut -c1-200
for c in C5 C4 C3 C2; do
  BENCH_NO_OBSERVABLES=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 2>$O/r02s_$c.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), round(d['roofline']['frac'],3), {k:round(v,2) for k,v in d['stages_ms_per_step'].items() if v})"
done
