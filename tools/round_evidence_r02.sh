#!/bin/bash
# Round-2 evidence: bench-step launch lists for c1/c2/c3/c4p6 (cold, serialised;
# shares matter) and ncu --set full of each config's dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02}
for cfg in c1 c2 c3 c4p6; do
  python bench.py --only --config $cfg --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench_$cfg.csv \
      python bench.py --only --config $cfg --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu_list_$cfg.log 2>&1
  echo "list $cfg rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 -o gpurun_out/${TAG}_c1_apply_full \
    python tools/prof_apply.py c1 > gpurun_out/${TAG}_ncu_c1.log 2>&1; echo "c1 full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_wsplit -s 3 -c 2 -o gpurun_out/${TAG}_c2_wsplit_full \
    python tools/prof_step.py c2 > gpurun_out/${TAG}_ncu_c2.log 2>&1; echo "c2 full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_big -s 3 -c 2 -o gpurun_out/${TAG}_c3_big_full \
    python tools/prof_step.py c3 > gpurun_out/${TAG}_ncu_c3.log 2>&1; echo "c3 full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_lowp -s 2 -c 1 -o gpurun_out/${TAG}_c4p6_lowp_full \
    python tools/prof_c4.py c4p6 > gpurun_out/${TAG}_ncu_c4.log 2>&1; echo "c4 full rc=$?"
ls gpurun_out/${TAG}_*
