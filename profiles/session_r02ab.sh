#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 2 --nccl-reserve 8 4 2 > gpurun_out/r02ab_split.txt 2>&1
timeout 900 python profiles/split_sustained.py --dims 16 16 16 4 --mask 8 --secs 1.0 --rounds 2 --nccl-reserve 8 4 2 > gpurun_out/r02ab_split_p8.txt 2>&1
cat gpurun_out/r02ab_split.txt gpurun_out/r02ab_split_p8.txt
