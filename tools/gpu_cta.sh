#!/bin/bash
# CTA-path (configs 2, 3) iteration: parity, timings, env-var A/B switches.
cd "$(dirname "$0")/.."
bash tools/gpu_quick.sh
for c in ${CONFIGS:-c2 c3}; do
  for v in ${ENVS}; do echo "== $c $v"; env $v=1 timeout 300 python tools/time_parts.py $c 2>&1 | grep -E "fused|apply cached|residual \(\+cache"; done
done
