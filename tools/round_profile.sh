#!/bin/bash
# Round-end evidence: default bench line, reference arm, launch list of the
# default bench, and a full ncu capture of the dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain_b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c1.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_b2.log 2>&1; echo "list rc=$?"
python tools/prof_apply.py c1 > gpurun_out/plain_apply.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 -o gpurun_out/prof_c1_apply_full \
    python tools/prof_apply.py c1 > gpurun_out/ncu_apply_full.log 2>&1; echo "full rc=$?"
