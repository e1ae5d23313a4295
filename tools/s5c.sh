#!/bin/bash
# Tucker part of a 64-plane slab at C5 / C4: FP64 DMMA (k_tucker_gemm_res) vs the
# Ozaki-split int8 tcgen05 GEMM (RSB200_TUCKER_OZ = slices)
O=gpurun_out
rm -f $O/s5c.log
for c in C5 C4; do
  for z in 0 7 6; do
    echo "== $c TUCKER_OZ=$z" >> $O/s5c.log
    RSB200_TUCKER_OZ=$z timeout 300 python tools/one_tucker.py $c 64 >> $O/s5c.log 2>&1
  done
done
cat $O/s5c.log
