timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python scripts/run_gemm.py
timeout 900 python scripts/run_config.py c5 2 2>&1 | grep "rep 1\|OK\|MISM"
timeout 900 python scripts/run_config.py c3 2 2>&1 | grep "rep 1\|OK\|MISM"
