#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "random_split" > gpurun_out/r02ad_fuzz.log 2>&1
echo "fuzz rc=$?"
tail -5 gpurun_out/r02ad_fuzz.log
