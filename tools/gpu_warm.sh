cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum -k regex:k_warp python tools/prof_apply.py c1 > gpurun_out/ncu_warm_c1.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "c4 or fused or residual" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for c in c4p2 c4p4 c4p6; do echo "== $c"; timeout 300 python tools/time_parts.py $c 2>&1 | grep -E "fused"; done
tail -2 gpurun_out/q_pytest.log
grep -E "k_warp|duration|cycles_active|dmma|bytes" gpurun_out/ncu_warm_c1.log | head -60
