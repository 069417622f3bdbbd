#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" > gpurun_out/r02v_fused.log 2>&1
echo "fused rc=$?"
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -s -k "timeout" > gpurun_out/r02v_timeout.log 2>&1
echo "timeout rc=$?"
tail -3 gpurun_out/r02v_fused.log; grep -E "waited|passed|failed|Error" gpurun_out/r02v_timeout.log | head
