#!/bin/bash
# round 2, session i: launch list of split (self-halo) applies vs unsplit, M5 fp16, peer and NCCL
mkdir -p gpurun_out
for tr in peer nccl; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_split_$tr.csv \
  python profiles/run_split.py --mask 8 --transport $tr --variant 10 --reps 4 > gpurun_out/r02i_split_$tr.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_nosplit.csv \
  python profiles/run_split.py --mask 0 --variant 10 --reps 4 > gpurun_out/r02i_nosplit.log 2>&1
echo done
