python scripts/time_dct.py 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "dct or ttm or reconstruct" 2>&1 | tail -1
