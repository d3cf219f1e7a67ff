#!/bin/bash
# Precise A/B of library builds on bench.py (default config c1, or CFG=...):
# 10 timed steps, twice per build.  VARIANTS="x y" -> paper_2412_13733_b200/libhpg_b200_<x>.so
cd $GRAFT_REPO_ROOT
for v in default ${VARIANTS}; do
  lib=""; [ "$v" != default ] && lib=$PWD/paper_2412_13733_b200/libhpg_b200_$v.so
  for rep in 1 2; do
    HPG_LIB=$lib python bench.py --config ${CFG:-c1} --rule ${RULE:-gauss} --steps ${STEPS:-10} --warmup 3 --e2e-steps 0 --no-cpu-baseline | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['value'], d['roofline']['avg_launch_us'])"
  done
done
