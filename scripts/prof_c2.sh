#!/bin/bash
# c2 step: launch list (ncu, serialised) + one full capture of the kernel matched by $KREGEX
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/run_step.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/run_step.py > gpurun_out/ncu_list.log 2>&1
echo "list exit $?"
if [ -n "$KREGEX" ]; then
  ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${KSKIP:-1} -c 1 -o gpurun_out/prof_$KNAME python scripts/run_step.py > gpurun_out/ncu_full.log 2>&1
  echo "full exit $?"
fi
python scripts/launch_summary.py gpurun_out/launches_c2.csv
