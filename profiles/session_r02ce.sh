#!/bin/bash
# round 2, session ce: fp16 ring epilogue with x * (1/s) instead of the IEEE division (CD_RING_EXP=8), same-box A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02ce_recip.txt
for e in 0 8 0 8; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
done
cat $O
