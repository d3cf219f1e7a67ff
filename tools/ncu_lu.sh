set -e
python tools/prof_precond.py c1 > gpurun_out/pp_c1.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lu -c 2 -o gpurun_out/ncu_lu_c1 python tools/prof_precond.py c1 > gpurun_out/ncu_lu.log 2>&1
