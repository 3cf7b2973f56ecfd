#!/bin/bash
# quick functional pass of bench.py variants on one GPU (logs in gpurun_out/)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c1}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 2 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c exit $?"; tail -c 3000 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
if [ -n "$SHARDED" ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 bench.py --sharded --config ${SHARDED} --steps 3 --warmup 2 > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err
  echo "sharded exit $?"; cat gpurun_out/bench_sharded.json; tail -5 gpurun_out/bench_sharded.err
fi
