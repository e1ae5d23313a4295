#!/bin/bash
# Round-2 profiling pass (run on the GPU box from the repo root): bench lines at
# every config (C5 = the default command, with the CPU baseline leg), reference
# arm, launch list of the default command and ncu --set full captures of the
# top kernels.  Numbers printed by runs under ncu are never bench values.
TAG=${TAG:-r02}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/${TAG}_smi.txt
nproc >> $O/${TAG}_smi.txt; free -g >> $O/${TAG}_smi.txt
# SASS evidence of the Blackwell paths (tcgen05 MMA, TMEM loads, bulk copies) and the FP64 tensor path
cuobjdump -sass paper_1606_09218_b200/librsb200.so > /tmp/rsb200.sass 2>/dev/null
for m in UTCIMMA LDTM UBLKCP UTMALDG DMMA LDGSTS; do echo "$m $(grep -c "$m" /tmp/rsb200.sass)"; done > $O/${TAG}_sass_counts.txt
python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.txt 2>&1
python bench.py > $O/${TAG}_bench_C5.json 2> $O/${TAG}_bench_C5.err
RSB200_TUCKER_OZ=0 python bench.py --no-cpu-baseline > $O/${TAG}_bench_C5_dmma_tucker.json 2> $O/${TAG}_bench_C5_dmma_tucker.err
for c in C4 C3 C2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference_C5.json 2> $O/${TAG}_ref.err
# launch list of the default command's step (ordinary streams: ncu cannot replay
# on the green-context side stream)
RSB200_SIDE_SMS=0 BENCH_NO_OBSERVABLES=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_C5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_launch.log 2>&1
# full captures (one launch of each top kernel, after the warm-up steps)
RSB200_SIDE_SMS=0 BENCH_NO_OBSERVABLES=1 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_short_mma|k_tucker_gemm_res|k_oz_res|k_oz_rowslice|k_core_h|k_syrk_part" -s 36 -c 10 -f -o $O/${TAG}_full_C5 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_C5.log 2>&1
summarise() {  # .ncu-rep files are tens of MB (gpurun_out/ is capped at 64 MiB): keep the tables
  python tools/ncu_summary.py $O/${TAG}_full_$1.ncu-rep > $O/${TAG}_ncu_summary_$1.md 2>&1
  ncu -i $O/${TAG}_full_$1.ncu-rep --page raw --csv > $O/${TAG}_ncu_raw_$1.csv 2>/dev/null
  rm -f $O/${TAG}_full_$1.ncu-rep
}
summarise C5
for c in C4 C3; do
  RSB200_SIDE_SMS=0 BENCH_NO_OBSERVABLES=1 timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"k_short_mma|k_tucker_gemm_res|k_tucker_apply|k_syrk_part" -s 21 -c 3 -f -o $O/${TAG}_full_$c \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_$c.log 2>&1
  summarise $c
done
RSB200_SIDE_SMS=0 BENCH_NO_OBSERVABLES=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_short_mma|k_tucker_apply|k_syrk_part" -s 21 -c 3 -f -o $O/${TAG}_full_C2 \
  python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_C2.log 2>&1
summarise C2
python tools/launch_shares.py $O/${TAG}_launches_C5.csv > $O/${TAG}_launch_shares_C5.md 2>&1
gzip -f $O/${TAG}_launches_C5.csv
