# End-of-round refresh: bench line, c2 launch list, reduce-kernel capture, configs at full size, tests, smoke.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_step.py > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svd_reduce_kernel --launch-skip 1 -c 1 -o gpurun_out/reduce_full python scripts/run_reduce.py > gpurun_out/ncu_full.log 2>&1
for c in c1 c3 c4; do timeout 1200 python scripts/run_config.py $c > gpurun_out/config_$c.log 2>&1; done
timeout 900 python scripts/run_config.py c5 2 > gpurun_out/config_c5.log 2>&1
timeout 900 python scripts/run_config.py c5 2 tol > gpurun_out/config_c5tol.log 2>&1
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
