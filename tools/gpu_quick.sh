#!/bin/bash
# Quick GPU iteration: parity subset + per-piece timings for the given configs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for c in ${CONFIGS:-c1}; do echo "== $c"; timeout 300 python tools/time_parts.py $c; done > gpurun_out/q_parts.log 2>&1
tail -3 gpurun_out/q_pytest.log; cat gpurun_out/q_parts.log
