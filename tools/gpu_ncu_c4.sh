#!/bin/bash
# ncu --set full of the config-4 low-degree kernel (tools/prof_c4.py CFG), report TAG
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/prof_c4.py ${CFG:-c4p2} > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_low}" -s ${SKIP:-2} -c ${COUNT:-1} \
    -o gpurun_out/prof_${TAG:-c4} python tools/prof_c4.py ${CFG:-c4p2} > gpurun_out/ncu_${TAG:-c4}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_${TAG:-c4}.log
