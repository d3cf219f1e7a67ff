cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
tail -3 gpurun_out/q_pytest.log
timeout 300 python tools/time_parts.py c1
for rule in gauss reference; do timeout 600 python bench.py --config c3 --rule $rule --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/r01b_all_c3_${rule}.json 2> gpurun_out/r01b_all_c3_${rule}.err; echo "c3 $rule rc=$?"; done
