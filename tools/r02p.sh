O=gpurun_out
rm -f $O/r02p_tucker.log
for bk in 16 32 16 32; do echo "BK=$bk" >> $O/r02p_tucker.log; RSB200_TUCKER_BK=$bk python tools/one_tucker.py C5 64 >> $O/r02p_tucker.log 2>&1; RSB200_TUCKER_BK=$bk python tools/one_tucker.py C4 64 >> $O/r02p_tucker.log 2>&1; done
cat $O/r02p_tucker.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_large.py -q -k "not C3" > $O/r02p_pytest.log 2>&1
tail -4 $O/r02p_pytest.log | cut -c1-200
