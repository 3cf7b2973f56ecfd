#!/bin/bash
# Round-2 (late) evidence: c2 launch list of the pruned step and ncu --set full
# captures of its kernels.  Outputs in gpurun_out/r2b/.
cd "$(dirname "$0")/.."
O=gpurun_out/r2b
mkdir -p $O
python scripts/run_step.py > $O/plain_step.log 2>&1 || { echo "plain step failed"; tail -5 $O/plain_step.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python scripts/run_step.py > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_c2.csv > $O/launches_c2_summary.txt 2>&1
cat $O/launches_c2_summary.txt
for k in ${KERNELS:-svd_reduce_kernel dct1024_kernel svd_bulge_kernel svd_bisect_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-1} -c 1 -f -o $O/prof_$k python scripts/run_step.py > /dev/null 2>&1
  echo "ncu $k $?"
  python scripts/ncu_summary.py $O/prof_$k.ncu-rep "c2 pruned step: $k (ncu --set full --clock-control none)" > $O/${k}_summary.txt 2>&1
done
