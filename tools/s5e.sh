#!/bin/bash
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "oz_gemm or tucker_gemm" > $O/s5e_pytest.txt 2>&1
tail -3 $O/s5e_pytest.txt
rm -f $O/s5e.log
for d in 128 144; do
  echo "== C5 DBG=$d" >> $O/s5e.log
  RSB200_OZ_DBG=$d timeout 120 python tools/one_tucker.py C5 64 2>&1 | tail -3 >> $O/s5e.log
done
cat $O/s5e.log
