#!/bin/bash
# Round-2 final evidence (tag r02c): GPU tests, smoke, both bench arms, bench-step
# launch lists (cold, serialised; shares matter) and ncu --set full of the kernels
# changed since r02a: the streaming cached apply (k_stream) and the row-per-thread LU (k_lu2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
for cfg in c1 c2 c3 c4p6; do
  python bench.py --only --config $cfg --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench_$cfg.csv \
      python bench.py --only --config $cfg --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu_list_$cfg.log 2>&1
  echo "list $cfg rc=$?"
done
python tools/prof_apply.py c1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stream -s 3 -c 1 -f -o gpurun_out/${TAG}_c1_stream_cold \
    python tools/prof_apply.py c1 > gpurun_out/${TAG}_ncu_c1_cold.log 2>&1; echo "c1 cold rc=$?"
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_stream -s 3 -c 1 -f -o gpurun_out/${TAG}_c1_stream_warm \
    python tools/prof_apply.py c1 > gpurun_out/${TAG}_ncu_c1_warm.log 2>&1; echo "c1 warm rc=$?"
python tools/prof_precond.py c1 > gpurun_out/${TAG}_precond_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_lu2 -s 1 -c 1 -f -o gpurun_out/${TAG}_c1_lu2 \
    python tools/prof_precond.py c1 > gpurun_out/${TAG}_ncu_lu2.log 2>&1; echo "lu2 rc=$?"
ls gpurun_out/${TAG}_* | head -40
