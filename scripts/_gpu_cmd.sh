timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python scripts/run_config.py c5 2 tol 2>&1 | tail -5
