O=gpurun_out
for w in 256 32 2048; do
for c in C5 C4; do
  RSB200_MMA_WAVES=$w BENCH_NO_OBSERVABLES=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02m_bench_${c}_w$w.json 2> $O/r02m_bench_${c}_w$w.err
done; done
for c in C3 C2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02m_bench_$c.json 2> $O/r02m_bench_$c.err
done
