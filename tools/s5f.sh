#!/bin/bash
O=gpurun_out
rm -f $O/s5f.log
for d in 0 1 3 4 7; do
  echo "== C5 TUCKER_OZ=7 DBG=$d" >> $O/s5f.log
  RSB200_OZ_DBG=$d RSB200_TUCKER_OZ=7 timeout 300 python tools/one_tucker.py C5 64 2>&1 | tail -1 >> $O/s5f.log
done
cat $O/s5f.log
