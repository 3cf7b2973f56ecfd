timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/run_step.py > gpurun_out/rs.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_step.py > /dev/null 2>&1; cat gpurun_out/rs.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','e2e','stages_ms']: print(k, d.get(k))"
