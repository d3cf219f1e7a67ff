#!/bin/bash
# parity of the touched paths + launch list + bench lines for the given configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
for cfg in ${CONFIGS:-c2}; do
  python tools/prof_step.py $cfg gauss > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv python tools/prof_step.py $cfg gauss > /dev/null 2>&1
  python tools/launches.py gpurun_out/launches_$cfg.csv > gpurun_out/launches_$cfg.txt 2>&1
  timeout 300 python bench.py --only --config $cfg --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$cfg.json'))
print('$cfg', 'value %.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline_frac'], 'kern %.3f'%d['roofline']['frac'], 'us %.2f'%d['roofline']['avg_launch_us'], 'res_ms %.4f'%d['res_ms_mean'])
" >> gpurun_out/quick_summary.txt 2>&1 || tail -3 gpurun_out/bench_$cfg.err >> gpurun_out/quick_summary.txt
done
tail -3 gpurun_out/pytest_q.log; cat gpurun_out/quick_summary.txt; for cfg in ${CONFIGS:-c2}; do echo "== $cfg"; cat gpurun_out/launches_$cfg.txt; done
