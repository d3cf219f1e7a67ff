#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench lines.  Output -> gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for cfg in ${BENCH_CONFIGS:-c1}; do
  timeout 600 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?" >> gpurun_out/bench_rc.log
done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/bench_rc.log; for f in gpurun_out/bench_*.json; do echo $f; cat $f; done
