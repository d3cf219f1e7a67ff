#!/bin/bash
# warm-cache launch lists (ncu --cache-control none) of prof_step for CONFIGS
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CONFIGS:-c2 c3}; do
  python tools/prof_step.py $cfg ${RULE:-gauss} > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
      --log-file gpurun_out/warm_$cfg.csv python tools/prof_step.py $cfg ${RULE:-gauss} > /dev/null 2>&1
  echo "== $cfg (warm)"; python tools/launches.py gpurun_out/warm_$cfg.csv
done
