# Full-size runs of every BASELINE config with the current kernels (energy-identity check).
mkdir -p gpurun_out
for c in c1 c3 c4; do echo "== $c"; timeout 1200 python scripts/run_config.py $c 2>&1 | grep -v Warning | tail -12; done > gpurun_out/configs_full.txt
echo "== c5" >> gpurun_out/configs_full.txt; timeout 900 python scripts/run_config.py c5 2 2>&1 | tail -5 >> gpurun_out/configs_full.txt
echo "== c5tol" >> gpurun_out/configs_full.txt; timeout 900 python scripts/run_config.py c5 2 tol 2>&1 | tail -5 >> gpurun_out/configs_full.txt
cat gpurun_out/configs_full.txt
