#!/bin/bash
# Every BASELINE config (both rules) through bench.py -> gpurun_out/all_<cfg>_<rule>.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rule in gauss reference; do
  for cfg in c0 c1 c2 c3 c4p2 c4p4 c4p6; do
    timeout 600 python bench.py --config $cfg --rule $rule --steps 5 --warmup 3 --e2e-steps 1 \
      > gpurun_out/all_${cfg}_${rule}.json 2> gpurun_out/all_${cfg}_${rule}.err
    echo "$cfg $rule rc=$?"
  done
done
