O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_short_mma.py -x -q -m "gpu and not slow" > $O/r02l_pytest.log 2>&1
tail -5 $O/r02l_pytest.log | cut -c1-250
for c in C4 C5; do
ncu --set full --clock-control none --import-source on -k regex:k_short_mma -s 2 -c 1 -f -o $O/r02l_mma_$c python tools/short_methods.py $c 64 mma > $O/r02l_ncu_$c.log 2>&1
done
ls -la $O/*.ncu-rep
