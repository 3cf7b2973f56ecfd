mkdir -p gpurun_out
python scripts/run_gemm.py
timeout 1200 python scripts/run_config.py c4 2 > gpurun_out/config_c4.log 2>&1; echo "exit $?" >> gpurun_out/config_c4.log
cat gpurun_out/config_c4.log
