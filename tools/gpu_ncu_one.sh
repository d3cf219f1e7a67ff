#!/bin/bash
# ncu --set full of kernels matching KREGEX in prof_step CFG (one GPU); TAG names the report
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/prof_step.py $CFG ${RULE:-gauss} > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-2} \
    -o gpurun_out/prof_${TAG} python tools/prof_step.py $CFG ${RULE:-gauss} > gpurun_out/ncu_${TAG}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
