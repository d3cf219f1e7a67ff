#!/bin/bash
# c4 iteration: parity + fused residual/apply timings, A/B library variants.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for c in c4p2 c4p4 c4p6; do
  echo "== $c default"; timeout 300 python tools/time_parts.py $c 2>&1 | grep -E "fused|no cache|apply from"
  for v in ${VARIANTS}; do echo "== $c $v"; HPG_LIB=$PWD/paper_2412_13733_b200/libhpg_b200_$v.so timeout 300 python tools/time_parts.py $c 2>&1 | grep fused; done
  echo "== $c old"; HPG_LOWP_OFF=1 timeout 300 python tools/time_parts.py $c 2>&1 | grep fused
done > gpurun_out/q_parts.log 2>&1
tail -3 gpurun_out/q_pytest.log; cat gpurun_out/q_parts.log
