O=gpurun_out
python -m pytest tests/test_gpu_short_l0.py -x -q > $O/r02b_pytest.log 2>&1
python tools/fused_bench.py C5 256 > $O/r02b_fused.log 2>&1
RSB200_LIB=gpurun_var/lib_gu4.so python tools/fused_bench.py C5 256 >> $O/r02b_fused.log 2>&1
python tools/one_short.py C5 256 0,1,2,3,4,5 > $O/r02b_short.log 2>&1
