#!/bin/bash
# round 2, session bj: M5 fp16 ring under sustained (power-capped) load with the persistent grid capped below 148 SMs
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bj_ring_sms.txt
for cap in 0 136 124 112 100 0; do
  echo "== CD_RING_SMS=$cap" >> $O
  CD_RING_SMS=$cap timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 3 >> $O 2>&1
done
cat $O
