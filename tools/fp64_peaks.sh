#!/bin/bash
# Measure FP64 peaks on the GPU box (DFMA loop, DMMA loop, cuBLAS DGEMM via torch)
# with nvidia-smi clocks sampled during the run.  Output: gpurun_out/fp64_peaks.log
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/fp64_clocks.csv &
SMI=$!
./tools/fp64_peaks > gpurun_out/fp64_peaks.log 2>&1
python - >> gpurun_out/fp64_peaks.log 2>&1 <<'EOF'
import torch, time, json
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"cublas_dgemm_tflops_burst": 2 * n**3 / best * 1e-9, "ms": best}))
t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b); k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(json.dumps({"cublas_dgemm_tflops_sustained": 2 * n**3 * k / e0.elapsed_time(e1) * 1e-9, "iters": k}))
EOF
kill $SMI || true
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem --format=csv >> gpurun_out/fp64_peaks.log
