timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],2), 'reconstruct', d['reconstruct'])"
timeout 1200 python scripts/run_config.py c4 1 2>&1 | tail -4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/run_config.py c4 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/c4_launches.csv all | grep "unpack\|gemm"
