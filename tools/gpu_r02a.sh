#!/bin/bash
# Round-2 first GPU pass: full GPU suite (no -x), smoke, c1 bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench rc=$?" >> gpurun_out/bench_c1.err
tail -30 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_c1.json | head -c 1500; tail -3 gpurun_out/bench_c1.err
