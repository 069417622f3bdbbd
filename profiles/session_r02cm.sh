#!/bin/bash
# round 2, session cm: compressed ring (fp16, three matrices per stage) with two CTAs per SM: parity + A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CD_COMP_2CTA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compress" > gpurun_out/r02cm_parity.log 2>&1
echo "parity(2cta) rc=$?"; tail -2 gpurun_out/r02cm_parity.log
O=gpurun_out/r02cm_comp2.txt
for r in 1 2; do
 for c in 1 0; do
  echo "== CD_COMP_2CTA=$c" >> $O
  CD_COMP_2CTA=$c timeout 300 python profiles/run_compressed_ab.py --dims 16 16 16 32 --prec fp16 --secs 0.6 >> $O 2>&1
  CD_COMP_2CTA=$c timeout 300 python profiles/run_compressed_ab.py --dims 8 8 8 8 --prec fp16 --secs 0.4 >> $O 2>&1
 done
done
cat $O
