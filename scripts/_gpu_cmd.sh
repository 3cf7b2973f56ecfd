timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/time_reduce.py 2>&1 | tail -1
timeout 300 python scripts/probe_reduce.py 2>&1 | tail -1
timeout 300 python scripts/run_step.py 2>&1 | tail -1
