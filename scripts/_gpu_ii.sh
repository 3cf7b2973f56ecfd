timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_step.py > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/ls.txt; grep "bdvec\|backtr" gpurun_out/ls.txt
timeout 1200 python scripts/run_config.py c4 2 2>&1 | grep "stages\|rep 1"
