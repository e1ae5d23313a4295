O=gpurun_out
rm -f $O/r02r.log
for g in 1 4 8 16 32; do
  for c in C5 C4; do
  echo "GROUPS=$g $c" >> $O/r02r.log
  BENCH_GROUPS=$g BENCH_NO_OBSERVABLES=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 4 2>>$O/r02r.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), {k:round(v,1) for k,v in d['stages_ms_per_step'].items() if v})" >> $O/r02r.log
  done
done
cat $O/r02r.log; tail -5 $O/r02r.err
