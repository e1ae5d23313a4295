O=gpurun_out
rm -f $O/r02k_methods.log
timeout 900 python -m pytest tests/test_gpu_short_mma.py -x -q -m "gpu and not slow" > $O/r02k_pytest.log 2>&1
tail -3 $O/r02k_pytest.log | cut -c1-250
for c in C2 C3 C4 C5; do timeout 600 python tools/short_methods.py $c 64 mma >> $O/r02k_methods.log 2>&1; done
grep mma $O/r02k_methods.log
