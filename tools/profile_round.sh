#!/bin/bash
# Round profiling pass (run on the GPU box from the repo root): bench lines,
# reference arm, launch list and ncu --set full captures of the top kernels.
# Numbers printed by runs under ncu are never bench values.
TAG=${TAG:-r01f}
O=gpurun_out
python bench.py > $O/${TAG}_bench_C2.json 2> $O/${TAG}_bench_C2.err
for c in C3 C4 C5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference_C2.json 2> $O/${TAG}_ref.err
# launch list of the C2 step (ordinary streams: ncu cannot replay on the green-context side stream)
RSB200_SIDE_SMS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_launch.log 2>&1
# full captures (one launch each, after the warm-up steps)
RSB200_SIDE_SMS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gemm_plane|k_tucker_apply|k_syrk_part|k_short_dmma" -s 20 -c 4 -f -o $O/${TAG}_full_C2 \
  python bench.py --steps 1 --warmup 8 --no-cpu-baseline > $O/${TAG}_ncu_c2.log 2>&1
for c in C3 C4; do
  RSB200_SIDE_SMS=0 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_gemm_plane|k_short_dmma|k_tucker_gemm_res" -s 12 -c 3 -f -o $O/${TAG}_full_$c \
    python bench.py --config $c --steps 1 --warmup 8 --no-cpu-baseline > $O/${TAG}_ncu_$c.log 2>&1
done
RSB200_SIDE_SMS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_short_l0|k_gemm_plane|k_tucker_gemm_res" -s 8 -c 2 -f -o $O/${TAG}_full_C5 \
  python bench.py --config C5 --steps 1 --warmup 8 --no-cpu-baseline > $O/${TAG}_ncu_C5.log 2>&1
