#!/bin/bash
# round 2, session bm: M5 fp16 ring m9 decomposition under sustained load: no vector copies (1), no consumer math (2)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bm_ring_exp.txt
for e in 0 1 2 3 0; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 3 >> $O 2>&1
done
cat $O
