#!/bin/bash
# Round-2 evidence refresh on one B200: GPU suite, bench lines for every
# config (ours + reference arm), c2 launch list and ncu captures of the
# dominant kernels.  Everything lands in gpurun_out/ (copied to profiles/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 1200 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
for c in c2 c1 c3 c4 c5 c5t; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c $?"
done
for c in c2 c1 c3; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $O/ref_$c.json 2> $O/ref_$c.err; echo "ref $c $?"
done
python scripts/run_step.py > $O/plain_step.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python scripts/run_step.py > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_c2.csv > $O/launches_c2_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:svd_reduce_kernel -s 1 -c 1 -o $O/prof_reduce_c2 python scripts/run_step.py > /dev/null 2>&1; echo "ncu reduce $?"
ncu --set full --clock-control none --import-source on -k regex:dct1024 -s 1 -c 1 -o $O/prof_dct_c2 python scripts/run_step.py > /dev/null 2>&1; echo "ncu dct $?"
ncu --set full --clock-control none --import-source on -k regex:residual_gemm -s 1 -c 1 -o $O/prof_residual_c2 python scripts/run_step.py > /dev/null 2>&1; echo "ncu residual $?"
