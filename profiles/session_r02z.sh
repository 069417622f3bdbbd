#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests/test_sanitizers.py -q > gpurun_out/r02z5_san.log 2>&1
echo "sanitizers rc=$?"
tail -4 gpurun_out/r02z5_san.log
grep -E "Race reported|and Read|Write access|Error" gpurun_out/r02z5_san.log | head -10
