#!/bin/bash
# round 2, session bc: multi-RHS pipeline skeleton (no copies / no build / no MMA combinations)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bc_mrhs_skeleton.txt
for d in "8 8 8 8 24" "6 6 6 12 32"; do
 set -- $d
 for e in 0 12 13 14 15 3 6 10; do
  echo "exp=$e $(CD_MRHS_EXP=$e timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5)" >> $O
 done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> $O
cat $O
