#!/bin/bash
# Run the GPU suite (or a subset: pass pytest args) on the gpurun box; logs to gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${T:-900} python -m pytest ${TESTS:-tests} -m gpu -q -rf --durations=15 "$@" > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
tail -30 gpurun_out/pytest_gpu.txt
