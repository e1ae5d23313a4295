O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/r02i_smi.txt
nproc >> $O/r02i_smi.txt; free -g >> $O/r02i_smi.txt
for c in C5 C4 C3 C2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02i_bench_$c.json 2> $O/r02i_bench_$c.err
done
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r02i_pytest.log 2>&1
tail -3 $O/r02i_pytest.log
