#!/bin/bash
# Launch lists (gpu__time_duration) for the prof_step driver of several configs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CONFIGS:-c1 c4p6}; do
  python tools/prof_step.py $cfg ${RULE:-gauss} ${BLOCKS:-} > gpurun_out/plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
      python tools/prof_step.py $cfg ${RULE:-gauss} ${BLOCKS:-} > gpurun_out/ncu_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
