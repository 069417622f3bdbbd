#!/bin/bash
# round 2, session x: full verification -- build + smoke, the whole GPU suite, the N=2 bench path
# on one GPU (--same-gpu, peer transport, fused split), the default bench, launch list
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02x_smoke.log 2>&1
echo "smoke rc=$?"
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02x_gpu_suite.log 2>&1
echo "gpu suite rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 10 --warmup 3 --same-gpu > gpurun_out/r02x_bench_2rank.json 2> gpurun_out/r02x_bench_2rank.err
echo "2-rank bench rc=$?"
export CD_TUNE_CACHE=gpurun_out/r02x_tune_cache.txt
timeout 900 python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02x_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02x_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
tail -3 gpurun_out/r02x_gpu_suite.log; tail -3 gpurun_out/r02x_smoke.log
