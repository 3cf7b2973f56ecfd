mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1200 python scripts/run_config.py c4 2 2>&1 | grep "stages\|rep 1"
timeout 900 python scripts/run_config.py c3 2 2>&1 | grep "rep 1"
STARM_LQ_WARP=1 timeout 900 python scripts/run_config.py c3 2 2>&1 | grep "rep 1"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'reduce', round(d['roofline']['ms'],2), 'e2e', round(d['e2e']['value'],2), 'value', round(d['value'],2))"
STARM_LQ_WARP=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('LQ_WARP ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'])"
