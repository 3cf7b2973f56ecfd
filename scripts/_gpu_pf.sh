mkdir -p gpurun_out
python scripts/probe_reduce.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), d['step_ms'], 'stages', d['stages_ms'], 'reduce', round(d['roofline']['ms'],2), 'dct', round(d['roofline']['dct']['ms'],3), 'e2e', round(d['e2e']['value'],2))"
timeout 1200 python scripts/run_config.py c4 2 > gpurun_out/config_c4.log 2>&1; echo "exit $?" >> gpurun_out/config_c4.log
cat gpurun_out/config_c4.log
