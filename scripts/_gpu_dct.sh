mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "dct or ttm" > gpurun_out/pytest_dct.log 2>&1; tail -3 gpurun_out/pytest_dct.log
python scripts/time_dct.py
STARM_DCT_LEGACY=1 python scripts/time_dct.py
