#!/bin/bash
# Full ncu capture of selected kernels of the prof_step driver (1 GPU, small launch count).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-c1}
python tools/prof_step.py $CFG ${RULE:-gauss} > gpurun_out/plain_full_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_warp}" -s ${SKIP:-0} -c ${COUNT:-4} \
    -o gpurun_out/prof_${TAG:-$CFG} python tools/prof_step.py $CFG ${RULE:-gauss} > gpurun_out/ncu_full_$CFG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full_$CFG.log
