O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parallel.py -x -q -k "C4 or C5 or ranks" > $O/r02n_pytest.log 2>&1
tail -3 $O/r02n_pytest.log
for c in C5 C4; do
  BENCH_NO_OBSERVABLES=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02n_bench_$c.json 2> $O/r02n_bench_$c.err
done
