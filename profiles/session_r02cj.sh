#!/bin/bash
# round 2, session cj: soak of the multi-rank peer path on one GPU (time-sliced processes): 10 x 2-rank bench,
# 3 x 4-rank bench (Z2 x T2), multi-rank parity tests twice
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02cj_soak.txt
for i in $(seq 1 10); do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + i)) bench.py --gpus 2 --steps 10 --warmup 3 --same-gpu > gpurun_out/r02cj_b2_$i.json 2> gpurun_out/r02cj_b2_$i.err
  echo "2-rank run $i rc=$? $(grep -c 'cd status' gpurun_out/r02cj_b2_$i.err)" >> $O
done
for i in 1 2 3; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29720 + i)) bench.py --gpus 4 --steps 6 --warmup 3 --same-gpu --pgrid 1,1,2,2 > gpurun_out/r02cj_b4_$i.json 2> gpurun_out/r02cj_b4_$i.err
  echo "4-rank run $i rc=$?" >> $O
done
for i in 1 2; do
  timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/r02cj_mr_$i.log 2>&1
  echo "multirank tests $i rc=$? $(tail -1 gpurun_out/r02cj_mr_$i.log)" >> $O
done
cat $O
