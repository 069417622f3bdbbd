#!/bin/bash
# round 2, session y: compressed-links TMA ring: parity, sanitizers, speed vs full links and vs the fine-grained kernel
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compressed" > gpurun_out/r02y_parity.log 2>&1
echo "parity rc=$?"
timeout 900 python -m pytest tests/test_sanitizers.py -q -x -k "compressed" > gpurun_out/r02y_san.log 2>&1
echo "san rc=$?"
for d in "16 16 16 32 fp16 24" "8 8 8 8 fp32 24" "8 8 8 8 fp16 24" "6 6 6 12 fp32 32" "6 6 6 12 fp16 32"; do
 set -- $d
 timeout 300 python profiles/run_compressed_ab.py --dims $1 $2 $3 $4 --prec $5 --nvec $6 >> gpurun_out/r02y_comp.txt 2>&1
 CD_COMP_RING=0 timeout 300 python profiles/run_compressed_ab.py --dims $1 $2 $3 $4 --prec $5 --nvec $6 --secs 0.5 | grep compressed | head -1 >> gpurun_out/r02y_comp.txt 2>&1
done
tail -3 gpurun_out/r02y_parity.log; cat gpurun_out/r02y_comp.txt
