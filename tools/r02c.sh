O=gpurun_out
python tools/one_short.py C5 64 > $O/r02c_plain.log 2>&1 && python tools/one_tucker.py C5 64 >> $O/r02c_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_short_l0|k_tucker_gemm_res" -c 2 -f -o $O/r02c_full python tools/fused_bench.py C5 64 > $O/r02c_ncu.log 2>&1
