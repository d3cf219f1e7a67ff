#!/bin/bash
# config 4: parity of the low-degree paths, then tiled (k_lowt) vs untiled (k_lowp) bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/lowt_ab.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "${PYTEST_K:-c4 or lowp or small or golden}" > gpurun_out/pytest_lowt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lowt.log
tail -3 gpurun_out/pytest_lowt.log
for cfg in ${CONFIGS:-c4p2 c4p4 c4p6}; do
  for v in tiled untiled; do
    if [ $v = untiled ]; then export HPG_LOWP_UNTILED=1; else unset HPG_LOWP_UNTILED; fi
    timeout 300 python bench.py --only --config $cfg --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${cfg}_$v.json 2> gpurun_out/bench_${cfg}_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_$v.json'))
print('$cfg $v', 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'us %.2f'%d['roofline']['avg_launch_us'])
" >> gpurun_out/lowt_ab.txt 2>&1 || tail -3 gpurun_out/bench_${cfg}_$v.err >> gpurun_out/lowt_ab.txt
  done
done
unset HPG_LOWP_UNTILED
cat gpurun_out/lowt_ab.txt
