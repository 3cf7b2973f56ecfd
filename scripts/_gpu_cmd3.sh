for per in 2 4 6 8 16; do
STARM_BISECT_SIDE_PER_SM=$per timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('per', $per, 'ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'])"
done
