#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_self and nccl" > gpurun_out/r02ae_parity.log 2>&1
echo "parity rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ae_split_nccl.csv \
  python profiles/run_split.py --mask 8 --transport nccl --variant 10 --reps 3 > /dev/null 2>&1
timeout 900 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 2 --nccl-reserve 8 4 > gpurun_out/r02ae_split.txt 2>&1
tail -2 gpurun_out/r02ae_parity.log; grep round gpurun_out/r02ae_split.txt
