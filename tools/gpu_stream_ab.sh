#!/bin/bash
# A/B of the streaming cached apply (hpg_stream.cuh) on config 1: parity subset, then bench per variant.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-c1}" > gpurun_out/s_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s_pytest.log
run() {  # label, lib, extra env
  for rep in 1 2; do
    env HPG_LIB=$2 $3 python bench.py --config ${CFG:-c1} --rule ${RULE:-gauss} --steps ${STEPS:-10} --warmup 3 --e2e-steps 0 --no-cpu-baseline --only | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'])"
  done
}
run nostream "" HPG_NO_STREAM=1
run default "" HPG_X=0
for v in ${VARIANTS}; do run $v $PWD/paper_2412_13733_b200/libhpg_b200_$v.so HPG_X=0; done
