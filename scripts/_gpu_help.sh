STARM_BULGE_HELPERS=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for h in 0 1 2; do
STARM_BULGE_HELPERS=$h python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('helpers $h ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'])"
done
