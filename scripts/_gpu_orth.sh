mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python scripts/run_config.py c4 2 2>&1 | tail -8
timeout 900 python scripts/run_config.py c3 2 2>&1 | tail -4
timeout 900 python scripts/run_config.py c5 2 tol 2>&1 | tail -4
