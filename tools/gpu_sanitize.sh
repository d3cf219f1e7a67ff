#!/bin/bash
# compute-sanitizer over the entry points (tools/sanitize_driver.py); TOOL=memcheck|racecheck|synccheck
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/sanitize_driver.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
for tool in ${TOOLS:-memcheck}; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --kernel-name-exclude regex:at:: --print-limit 50 \
    python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -6 gpurun_out/sanitize_$tool.log
done
tail -3 gpurun_out/sanitize_plain.log
