mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "bitwise or degenerate" 2>&1 | tail -1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/run_config.py c4 1 > gpurun_out/c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/c4_launches.csv all > gpurun_out/c4_launches_summary.txt 2>&1
head -14 gpurun_out/c4_launches_summary.txt
