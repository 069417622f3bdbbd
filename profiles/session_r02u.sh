#!/bin/bash
# round 2, session u: per-rank view of M5 at 8 GPUs (local 16^3x4, half the sites on a T face):
# unsplit vs fused vs unfused split, sustained; ncu launch lists
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python profiles/split_sustained.py --dims 16 16 16 4 --mask 8 --secs 1.0 --rounds 2 > gpurun_out/r02u_p8.txt 2>&1
timeout 600 python profiles/split_sustained.py --dims 16 16 8 8 --mask 12 --secs 1.0 --rounds 2 > gpurun_out/r02u_p8zt.txt 2>&1
for fu in 1 0; do
CD_FUSE_SPLIT=$fu timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02u_split_p8_$fu.csv \
  python profiles/run_split.py --dims 16 16 16 4 --mask 8 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02u_nosplit_p8.csv \
  python profiles/run_split.py --dims 16 16 16 4 --mask 0 --variant 10 --reps 3 > /dev/null 2>&1
cat gpurun_out/r02u_p8.txt gpurun_out/r02u_p8zt.txt
