O=gpurun_out
rm -f $O/r02k_methods.log
RSB200_MMA_BUILD=1 timeout 900 python -m pytest tests/test_gpu_short_mma.py -x -q -m "gpu and not slow" > $O/r02k_pytest.log 2>&1
tail -3 $O/r02k_pytest.log | cut -c1-250
for c in C2 C3 C4 C5; do
 for b in 0 1; do echo "BUILD=$b" >> $O/r02k_methods.log; RSB200_MMA_BUILD=$b timeout 600 python tools/short_methods.py $c 64 mma >> $O/r02k_methods.log 2>&1; done
done
grep -E "mma|BUILD" $O/r02k_methods.log | cut -c1-150
