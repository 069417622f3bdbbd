#!/bin/bash
# round 2, session cb: repeat the 2-rank same-GPU bench (peer transport, time-sliced processes) to see how often it times out
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2 3 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29670 + i)) bench.py --gpus 2 --steps 10 --warmup 3 --same-gpu > gpurun_out/r02cb_bench_2rank_$i.json 2> gpurun_out/r02cb_bench_2rank_$i.err
  echo "run $i rc=$?"
  grep -o '"variant": "[a-z0-9_]*"' gpurun_out/r02cb_bench_2rank_$i.json | head -1
  grep -o "cd status -7" gpurun_out/r02cb_bench_2rank_$i.err | head -1
done
