timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python scripts/probe_reduce.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'reduce', round(d['roofline']['ms'],2))"
timeout 900 python scripts/run_config.py c3 2 2>&1 | grep "rep 1"
