#!/bin/bash
# Launch lists + full ncu captures of the c2 / c3 step kernels (gauss rule).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in c2 c3; do
  python tools/prof_step.py $cfg gauss > gpurun_out/plain_$cfg.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
      python tools/prof_step.py $cfg gauss > gpurun_out/ncu_list_$cfg.log 2>&1
  echo "$cfg list rc=$?"
done
# full capture of the third (warm) iteration's kernels
for cfg in c2 c3; do
  ncu --set full --clock-control none --import-source on -k "regex:k_cta|k_uside_pt|k_hat_gather|k_warp" -s 12 -c 6 \
      -o gpurun_out/prof_r02_$cfg python tools/prof_step.py $cfg gauss > gpurun_out/ncu_full_$cfg.log 2>&1
  echo "$cfg full rc=$?"
done
ls -la gpurun_out/
