timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for L in 1 0; do
rm -f build/svd_f64.o paper_2605_16058_b200/libstarm.so; make -j8 NVEXTRA="-DSTARM_LOCAL_HOUSE=$L" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_step.py > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/ls.txt; echo "LOCAL_HOUSE=$L $(grep bulge gpurun_out/ls.txt)"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'])"
done
