#!/bin/bash
# round 2, session bs: decomposition of the other ring configs (fp32 M3 m3, fp32 M4 m3, fp16 M4 m3) under sustained load
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bs_ring_exp.txt
for e in 0 1 2 0; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp32 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 16 --nvec 24 --prec fp32 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
done
cat $O
