cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c1 c2 c3 c4p2 c4p4 c4p6; do echo "== $c"; timeout 300 python tools/time_parts.py $c; done > gpurun_out/parts.log 2>&1
for c in c2 c3 c4p6; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
python tools/prof_apply.py c1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 -o gpurun_out/c1_apply_full python tools/prof_apply.py c1 > gpurun_out/ncu_full.log 2>&1
echo done
