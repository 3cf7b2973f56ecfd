nproc; uptime
for i in 1 2 3 4; do
STARM_BENCH_NO_SMI=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nosmi', d['step_ms'])"
done
uptime
