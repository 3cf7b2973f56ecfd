# quick GPU iteration: tests, reduce phase split, bench
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python scripts/probe_reduce.py
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','e2e','stages_ms']: print(k, d.get(k))
print('reduce', d['roofline']['ms'], d['roofline']['frac'])"
