#!/bin/bash
# K-chunk promotion sweep (GPU box): cfg3 step time per (VNT_TC_KFIRST, VNT_TC_KCHUNK).
for cfg in ${CFGS:-"1024 0" "1024 256"}; do
  set -- $cfg
  VNT_TC_KFIRST=$1 VNT_TC_KCHUNK=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra \
    > gpurun_out/sweep_kf$1_kc$2.json 2> gpurun_out/sweep_kf$1_kc$2.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/sweep_kf$1_kc$2.json").read().strip().splitlines()[-1])
print("kfirst $1 kchunk $2", round(d["value"]), "samples/s", round(d["ms_per_step"], 3), "ms/step frac",
      round(d["roofline"]["frac"], 3))
PY
done
