#!/bin/bash
# A/B of 32-wide x3 tiles in the fused short kernel (RSB200_MMA_T3=32: three CTAs per SM)
O=gpurun_out
rm -f $O/s5l.log
for c in C5 C4 C3 C2; do
  for t in 64 32; do
    echo "== $c T3=$t" >> $O/s5l.log
    RSB200_MMA_T3=$t timeout 600 python tools/short_methods.py $c 64 l0,mma 2>&1 | tail -1 >> $O/s5l.log
  done
done
RSB200_MMA_T3=32 timeout 900 python -m pytest tests -m gpu -x -q -k "short_mma or edges or parity" > $O/s5l_pytest.txt 2>&1
tail -2 $O/s5l_pytest.txt
cat $O/s5l.log
