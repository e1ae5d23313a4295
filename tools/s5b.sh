#!/bin/bash
O=gpurun_out
rm -f $O/s5b.log
for c in C5 C4; do
  for d in 0 1 2; do
    echo "== $c DBG=$d" >> $O/s5b.log
    RSB200_MMA_DBG=$d timeout 600 python tools/short_methods.py $c 64 mma >> $O/s5b.log 2>&1
  done
done
cat $O/s5b.log
