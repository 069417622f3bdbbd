#!/bin/bash
# round 2, session ac: per-rank view of M5 strong scaling on one GPU (local volumes of N = 1, 2, 4, 8;
# the T faces routed through the fused split apply with a self exchange)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for d in "16 16 16 32" "16 16 16 16" "16 16 16 8" "16 16 16 4"; do
  timeout 300 python profiles/split_sustained.py --dims $d --mask 8 --secs 0.8 --rounds 2 | sed "s/^/L=${d// /x} T: /" >> gpurun_out/r02ac_scaling.txt
done
timeout 300 python profiles/split_sustained.py --dims 16 16 8 8 --mask 12 --secs 0.8 --rounds 2 | sed "s/^/L=16x16x8x8 ZT: /" >> gpurun_out/r02ac_scaling.txt
cat gpurun_out/r02ac_scaling.txt
