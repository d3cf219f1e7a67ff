#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c4p6 c4p4; do
python tools/prof_c4.py $c > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 -k regex:k_lowp -s 2 -c 1 -o gpurun_out/prof_$c python tools/prof_c4.py $c > gpurun_out/ncu_$c.log 2>&1
done
for c in c4p2 c4p4 c4p6; do echo "== $c"; timeout 300 python tools/time_parts.py $c 2>&1 | grep -E "fused"; done
