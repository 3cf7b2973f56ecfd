timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/run_c3_step.py > gpurun_out/c3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/run_c3_step.py > /dev/null 2>&1; cat gpurun_out/c3.log
timeout 300 python scripts/run_step.py > gpurun_out/rs.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_step.py > /dev/null 2>&1; cat gpurun_out/rs.log
