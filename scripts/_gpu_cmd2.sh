for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nvml', d['step_ms'], d['clocks'], d['value'])"
done
