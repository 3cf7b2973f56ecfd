#!/bin/bash
# inverse-iteration threads per SM sweep on c4 (launch list per setting)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/run_wl_step.py c4 > gpurun_out/plain_ii.log 2>&1 || exit 1
for v in 128 512 1024; do
  STARM_II_PER_SM=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:svd_bdvec --csv --log-file gpurun_out/ii_$v.csv python scripts/run_wl_step.py c4 > /dev/null 2>&1
  echo "== $v"; python scripts/launch_summary.py gpurun_out/ii_$v.csv all 2>/dev/null | tail -2
done
