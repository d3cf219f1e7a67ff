#!/bin/bash
# ncu --set full of the config-1 cached apply (k_stream), cold (default cache control) and warm L2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_apply.py c1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_stream}" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG:-stream}_cold -f python tools/prof_apply.py c1 > gpurun_out/ncu_${TAG:-stream}_cold.log 2>&1
echo "cold rc=$?"
ncu --set full --clock-control none --cache-control none --import-source on -k "regex:${KREGEX:-k_stream}" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG:-stream}_warm -f python tools/prof_apply.py c1 > gpurun_out/ncu_${TAG:-stream}_warm.log 2>&1
echo "warm rc=$?"
