#!/bin/bash
# Round evidence in one GPU call: default bench line, reference arm, the
# bench's launch list, full ncu of the dominant kernels (c1 cached apply,
# c4 p=6 single-pass residual), and every BASELINE config through bench.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01b}
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_plain_b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench_c1.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu_b2.log 2>&1; echo "list rc=$?"
python tools/prof_apply.py c1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 -o gpurun_out/${TAG}_c1_apply_full \
    python tools/prof_apply.py c1 > gpurun_out/${TAG}_ncu_apply_full.log 2>&1; echo "full rc=$?"
python tools/prof_c4.py c4p6 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_lowp -s 2 -c 1 -o gpurun_out/${TAG}_c4p6_lowp_full \
    python tools/prof_c4.py c4p6 > gpurun_out/${TAG}_ncu_lowp_full.log 2>&1; echo "lowp full rc=$?"
for rule in gauss reference; do
  for cfg in c0 c1 c2 c3 c4p2 c4p4 c4p6; do
    timeout 600 python bench.py --config $cfg --rule $rule --steps 5 --warmup 3 --e2e-steps 1 \
      > gpurun_out/${TAG}_all_${cfg}_${rule}.json 2> gpurun_out/${TAG}_all_${cfg}_${rule}.err
    echo "$cfg $rule rc=$?"
  done
done
