#!/bin/bash
# A/B timings: default library vs variants (HPG_LIB), for c1 apply and c4 fused entries.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for v in default ${VARIANTS}; do
  lib=""; [ "$v" != default ] && lib=$PWD/paper_2412_13733_b200/libhpg_b200_$v.so
  for c in ${CONFIGS:-c1 c4p2 c4p4 c4p6}; do
    echo "== $c $v"; HPG_LIB=$lib timeout 300 python tools/time_parts.py $c 2>&1 | grep -E "fused|apply cached"
  done
done > gpurun_out/q_parts.log 2>&1
tail -3 gpurun_out/q_pytest.log; cat gpurun_out/q_parts.log
