# quick GPU iteration: tests, reduce phase split, bench (twice: stability)
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
#timeout 300 python scripts/probe_reduce.py
for i in 1; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'steps', d.get('step_ms'), 'retries', d.get('alloc_retries'), 'stages', d['stages_ms'], 'dct', round(d['roofline']['dct']['ms'],3), 'reduce', round(d['roofline']['ms'],2), round(d['roofline']['frac'],3), 'clk', d['clocks'])"
done
