mkdir -p gpurun_out
python scripts/probe_reduce.py > gpurun_out/probe_plain.log 2>&1
make clean >/dev/null; make -j8 NVEXTRA=-DSTARM_PF_PROBE > /dev/null 2>&1
python scripts/probe_reduce.py > gpurun_out/probe_pf.log 2>&1
cat gpurun_out/probe_plain.log gpurun_out/probe_pf.log
