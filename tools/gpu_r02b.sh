#!/bin/bash
# full-size parity (new tests), krylov cost split, default bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_dropin.py -q -p no:cacheprovider --timeout 900 -k "full_size or grad_p2" > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 300 python tools/prof_krylov.py c1 > gpurun_out/prof_krylov.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?" >> gpurun_out/bench_default.err
tail -15 gpurun_out/pytest_full.log; cat gpurun_out/prof_krylov.log; tail -3 gpurun_out/bench_default.err
