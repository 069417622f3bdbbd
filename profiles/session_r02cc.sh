#!/bin/bash
# round 2, session cc: multi-rank bench (same GPU) after the count-based settle phase: 2 ranks x3, 4 ranks, 8 ranks
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2 3; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29680 + i)) bench.py --gpus 2 --steps 10 --warmup 3 --same-gpu > gpurun_out/r02cc_bench_2rank_$i.json 2> gpurun_out/r02cc_bench_2rank_$i.err
  echo "2 ranks run $i rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29690 bench.py --gpus 4 --steps 6 --warmup 3 --same-gpu --pgrid 1,1,2,2 > gpurun_out/r02cc_bench_4rank.json 2> gpurun_out/r02cc_bench_4rank.err
echo "4 ranks rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 8 --steps 4 --warmup 3 --same-gpu > gpurun_out/r02cc_bench_8rank.json 2> gpurun_out/r02cc_bench_8rank.err
echo "8 ranks rc=$?"
tail -c 300 gpurun_out/r02cc_bench_8rank.json
