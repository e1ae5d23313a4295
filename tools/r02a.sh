O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/r02a_smi.txt
nproc >> $O/r02a_smi.txt; free -g >> $O/r02a_smi.txt
for c in C5 C4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/r02a_bench_$c.json 2> $O/r02a_bench_$c.err
done
