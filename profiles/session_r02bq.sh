#!/bin/bash
# round 2, session bq: M5 fp16 ring m9 (gather4 producer) decomposition under sustained load
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bq_ring_exp.txt
for e in 0 2 4 6 0; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 3 >> $O 2>&1
done
cat $O
