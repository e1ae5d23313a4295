#!/bin/bash
# C5 step against the CTA-lifetime (RSB200_MMA_WAVES) and side-partition (RSB200_SIDE_SMS) knobs
O=gpurun_out
rm -f $O/s5k.log
run() {
  env "$@" timeout 600 python bench.py --config C5 --no-cpu-baseline --steps 6 > $O/s5k_tmp.json 2> $O/s5k_tmp.err
  python - "$*" <<'P' >> gpurun_out/s5k.log
import json, sys
try:
    d = json.loads(open("gpurun_out/s5k_tmp.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"], 2), {k: round(v, 1) for k, v in d["stages_ms_per_step"].items() if v})
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
}
export BENCH_NO_OBSERVABLES=1
run RSB200_MMA_WAVES=256
run RSB200_MMA_WAVES=64
run RSB200_MMA_WAVES=1024
run RSB200_SIDE_SMS=148
run RSB200_SIDE_SMS=132
run RSB200_SIDE_SMS=144
cat $O/s5k.log
