for i in 1 2; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), 'stages', d['stages_ms'], d['step_ms'][:4])"
done
