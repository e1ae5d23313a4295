O=gpurun_out
for c in C5 C4 C3 C2; do
  BENCH_NO_OBSERVABLES=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02n_bench_$c.json 2> $O/r02n_bench_$c.err
done
