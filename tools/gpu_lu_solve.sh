#!/bin/bash
# LU solve rewrite: parity of the preconditioner paths + per-config factor/apply timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_precond.py -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_lu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lu.log
tail -5 gpurun_out/pytest_lu.log
timeout 900 python tools/prof_precond.py ${CONFIGS:-c1 c2 c3 c4p4} > gpurun_out/prof_precond.log 2>&1; cat gpurun_out/prof_precond.log | grep -v Warning
