timeout 900 python -m pytest tests -m gpu -x -q -k "dct or ttm or tolerance" 2>&1 | tail -3
timeout 300 python scripts/run_step.py > gpurun_out/rs.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_step.py > /dev/null 2>&1; cat gpurun_out/rs.log
