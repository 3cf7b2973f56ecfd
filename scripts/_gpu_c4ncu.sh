mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/run_config.py c4 1 > gpurun_out/c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/c4_launches.csv > gpurun_out/c4_launches_summary.txt 2>&1
head -40 gpurun_out/c4_launches_summary.txt
