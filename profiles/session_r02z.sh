#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests/test_sanitizers.py -q -k "transport" > gpurun_out/r02z6_san.log 2>&1
echo "sanitizers rc=$?"
tail -4 gpurun_out/r02z6_san.log
grep -E "Race reported|and Read|Write access|Error" gpurun_out/r02z6_san.log | head -10
