#!/bin/bash
# round 2, session n: full GPU suite (parity, multi-rank, sanitizers, bench contract) + bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 3000 python -m pytest tests -q -m gpu -x > gpurun_out/r02n_gpu_suite.log 2>&1
echo "gpu suite rc=$?"
timeout 900 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
echo "bench rc=$?"
tail -5 gpurun_out/r02n_gpu_suite.log
