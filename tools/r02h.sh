O=gpurun_out
for c in C5 C4 C2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02h_bench_$c.json 2> $O/r02h_bench_$c.err
done
