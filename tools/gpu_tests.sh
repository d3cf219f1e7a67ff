#!/bin/bash
# full GPU test suite (or PYTEST_K subset); summary at the end
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_FILES} > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
grep -E "passed|failed|error" gpurun_out/pytest_all.log | tail -5; grep -E "^FAILED|^ERROR" gpurun_out/pytest_all.log | head -20
