#!/bin/bash
# ncu of the CTA-path kernels (configs 2 and 3): launch lists of the residual
# and apply, full capture of one cached apply launch each.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c2 c3; do
  timeout 300 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size python tools/prof_apply.py $c > gpurun_out/ncu_list_$c.log 2>&1
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_cta -s 3 -c 1 -o gpurun_out/prof_${c}_apply python tools/prof_apply.py $c > gpurun_out/ncu_full_$c.log 2>&1
done
echo done
