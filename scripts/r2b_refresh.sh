#!/bin/bash
# Round-2 (final) evidence refresh on one B200: GPU suite, bench lines for
# every config (ours + reference arm for c2/c1), launch lists (c2, c1, c3 with
# both bulge-chase variants, c4) and ncu --set full captures of the c2 step's
# kernels.  Everything lands in gpurun_out/r2b/ (summaries copied to profiles/).
cd "$(dirname "$0")/.."
O=gpurun_out/r2b
R=/tmp/r2b_ncu      # ncu reports stay on the box (gpurun_out is capped at 64 MiB): summaries only
mkdir -p $O $R
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt; tail -2 $O/pytest_gpu.txt
for c in ${CONFIGS:-c2 c1 c3 c4 c5 c5t}; do
  timeout 1200 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c $?"
done
for c in c2 c1; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $O/ref_$c.json 2> $O/ref_$c.err; echo "ref $c $?"
done
for c in c2 c1 c3 c4; do
  python scripts/run_wl_step.py $c > $O/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv python scripts/run_wl_step.py $c > /dev/null 2>&1
  python scripts/launch_summary.py $O/launches_$c.csv > $O/launches_${c}_summary.txt 2>&1
done
STARM_BULGE_CLUSTER=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_gmem_bulge.csv python scripts/run_wl_step.py c3 > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_c3_gmem_bulge.csv > $O/launches_c3_gmem_bulge_summary.txt 2>&1
for k in svd_reduce_kernel dct1024_kernel residual_gemm_kernel svd_bulge_kernel svd_bisect_kernel svd_bdvec_smem_kernel svd_backtransform_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f -o $R/prof_$k python scripts/run_step.py > /dev/null 2>&1
  echo "ncu $k $?"
  python scripts/ncu_summary.py $R/prof_$k.ncu-rep "c2 step: $k (ncu --set full --clock-control none)" > $O/${k}_summary.txt 2>&1
  python scripts/ncu_source_top.py $R/prof_$k.ncu-rep 16 > $O/${k}_source_top.txt 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -s 1 -c 1 -f -o $R/prof_gemm_c3 python scripts/run_gemm.py > /dev/null 2>&1
python scripts/ncu_summary.py $R/prof_gemm_c3.ncu-rep "c3-shaped dense transform: gemm_f64_kernel" > $O/gemm_c3_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_pers_kernel -s 1 -c 1 -f -o $R/prof_rec_gemm python scripts/run_reconstruct.py > /dev/null 2>&1
python scripts/ncu_summary.py $R/prof_rec_gemm.ncu-rep "c2 fused reconstruction GEMM (K = 64, ERR epilogue)" > $O/rec_gemm_summary.txt 2>&1
ls $O
