O=gpurun_out
rm -f $O/r02t.log
for mode in pipelined grouped prefetch; do
  for c in C5 C4; do
  echo "E2E=$mode $c" >> $O/r02t.log
  BENCH_E2E=$mode BENCH_NO_OBSERVABLES=1 timeout 900 python bench.py --config $c --no-cpu-baseline --steps 3 2>>$O/r02t.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1))" >> $O/r02t.log
  done
done
cat $O/r02t.log; tail -3 $O/r02t.err
