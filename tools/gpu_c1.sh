#!/bin/bash
# c1 apply-kernel iteration: parity, timings with/without PDL, fine-sampled ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
(echo "== c1 pdl"; timeout 300 python tools/time_parts.py c1; echo "== c1 nopdl"; HPG_NO_PDL=1 timeout 300 python tools/time_parts.py c1) > gpurun_out/q_parts.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/q_bench.json 2>gpurun_out/q_bench.err
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_warp -s 3 -c 1 -o gpurun_out/c1_apply_v2 python tools/prof_apply.py c1 > gpurun_out/ncu_v2.log 2>&1
tail -3 gpurun_out/q_pytest.log; cat gpurun_out/q_parts.log; python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print(d['value'],d['roofline']['frac'],d['roofline']['avg_launch_us'])"
