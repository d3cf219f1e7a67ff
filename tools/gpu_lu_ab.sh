#!/bin/bash
# A/B of the per-cell LU factor (k_lu) at config 1: variants x panel widths.
cd $GRAFT_REPO_ROOT
for v in default ${VARIANTS}; do
  lib=""; [ "$v" != default ] && lib=$PWD/paper_2412_13733_b200/libhpg_b200_$v.so
  for kb in ${KBS:-32 16 8}; do
    echo "== $v KB=$kb"; HPG_LIB=$lib HPG_LU_KB=$kb HPG_LU_PROF=1 python tools/prof_precond.py ${CFG:-c1} 2>&1 | grep -E "phases|factor" | cut -c1-250
  done
done
