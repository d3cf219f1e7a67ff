cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
SECONDS=0; python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$? wall ${SECONDS}s"
SECONDS=0; python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$? wall ${SECONDS}s"
python -c "
import json
d=json.load(open('gpurun_out/final_bench.json')); r=json.load(open('gpurun_out/final_ref.json'))
print('b200', d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'])
print('ref', r['value'], r['e2e'])
"
