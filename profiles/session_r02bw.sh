#!/bin/bash
# round 2, session bw: M5 fp16 ring m9 consumer decomposition (loads without FHFMA, no quantising epilogue)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bw_consumer.txt
for e in 0 2 8 16 24 0; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 3 >> $O 2>&1
done
cat $O
