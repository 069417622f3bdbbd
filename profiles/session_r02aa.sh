#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or halo_self" > gpurun_out/r02aa_parity.log 2>&1
echo "parity rc=$?"
timeout 900 python -m pytest tests/test_sanitizers.py -q -k "transport" > gpurun_out/r02aa_san.log 2>&1
echo "san rc=$?"
timeout 600 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 2 > gpurun_out/r02aa_split.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02aa_split_nccl.csv \
  python profiles/run_split.py --mask 8 --transport nccl --variant 10 --reps 3 > /dev/null 2>&1
tail -3 gpurun_out/r02aa_parity.log gpurun_out/r02aa_san.log | cat
