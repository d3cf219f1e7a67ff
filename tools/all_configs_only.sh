#!/bin/bash
# Every BASELINE config under both quadrature rules, each as the headline of its own
# bench.py --only run -> gpurun_out/<TAG>_all_<cfg>_<rule>.json (tools/summarize_all.py <TAG>)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02d}
for rule in gauss reference; do
  for cfg in c0 c1 c2 c3 c4p2 c4p4 c4p6; do
    timeout 900 python bench.py --only --config $cfg --rule $rule --steps 5 --warmup 3 --e2e-steps 2 \
      > gpurun_out/${TAG}_all_${cfg}_${rule}.json 2> gpurun_out/${TAG}_all_${cfg}_${rule}.err
    echo "$cfg $rule rc=$?"
  done
done
