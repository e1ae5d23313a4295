#!/bin/bash
# A/B of the x3-block skip in the fused short kernel (RSB200_MMA_SKIP)
O=gpurun_out
for c in C5 C4 C3 C2; do
  for s in 0 1; do  # 1 = skip unreachable x3 blocks
    echo "== $c SKIP=$s" >> $O/s5a.log
    RSB200_MMA_SKIP=$s timeout 600 python tools/short_methods.py $c 64 mma >> $O/s5a.log 2>&1
  done
done
python -m pytest tests -m gpu -x -q -k "short or mma or grid or large or reference" > $O/s5a_pytest.txt 2>&1
tail -3 $O/s5a_pytest.txt
cat $O/s5a.log
