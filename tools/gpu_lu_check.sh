#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_precond.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 900 -k "c3 or precond or slab" > gpurun_out/pytest_lu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lu.log
tail -30 gpurun_out/pytest_lu.log
timeout 600 python tools/prof_precond.py c3 > gpurun_out/prof_precond_c3.log 2>&1; tail -5 gpurun_out/prof_precond_c3.log
