#!/bin/bash
# launch lists of one workload step with the blocked / per-warp back-transformation
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=${C:-c3}
python scripts/run_wl_step.py $C > gpurun_out/plain_bt.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${C}_bt1.csv python scripts/run_wl_step.py $C > /dev/null 2>&1
STARM_BT_BLOCKED=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${C}_bt0.csv python scripts/run_wl_step.py $C > /dev/null 2>&1
echo "== blocked"; python scripts/launch_summary.py gpurun_out/launches_${C}_bt1.csv | head -12
echo "== per-warp"; python scripts/launch_summary.py gpurun_out/launches_${C}_bt0.csv | head -12
