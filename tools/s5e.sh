#!/bin/bash
O=gpurun_out
rm -f $O/s5e.log
for d in 128 136 137 139; do
  echo "== C5 DBG=$d" >> $O/s5e.log
  RSB200_OZ_DBG=$d timeout 300 python tools/one_tucker.py C5 64 2>&1 | tail -2 >> $O/s5e.log
done
cat $O/s5e.log
