mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/probe_reduce.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'reduce', round(d['roofline']['ms'],2), 'frac', round(d['roofline']['frac'],3), 'dct', round(d['roofline']['dct']['ms'],3), 'e2e', round(d['e2e']['value'],2), 'value', round(d['value'],2))"
timeout 900 python scripts/run_config.py c3 2 2>&1 | tail -3
