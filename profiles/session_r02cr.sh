#!/bin/bash
# round 2, session cr: ring m3 with two CTAs per SM (variant 11 for fp16 Nvec 24) vs ring m9; compressed ring 2-CTA re-check
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02cr_parity.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/r02cr_parity.log
O=gpurun_out/r02cr_ab.txt
timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 11 --secs 0.6 --rounds 4 >> $O 2>&1
timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 11 --secs 0.4 --rounds 3 >> $O 2>&1
for c in 1 0; do
  echo "== CD_COMP_2CTA=$c" >> $O
  CD_COMP_2CTA=$c timeout 300 python profiles/run_compressed_ab.py --dims 16 16 16 32 --prec fp16 --secs 0.6 >> $O 2>&1
done
cat $O
