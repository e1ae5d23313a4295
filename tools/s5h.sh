#!/bin/bash
# A/B of the grouped candidate search of the fused short kernel (RSB200_MMA_GROUP)
O=gpurun_out
rm -f $O/s5h.log
for g in 0 1; do
  echo "== C5 GROUP=$g" >> $O/s5h.log
  RSB200_MMA_GROUP=$g timeout 600 python tools/short_methods.py C5 64 l0,mma >> $O/s5h.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q -k "short_mma or reference_large or large or parity or edges" > $O/s5h_pytest.txt 2>&1
tail -3 $O/s5h_pytest.txt
cat $O/s5h.log
