#!/bin/bash
# round 2, session bp: gather4 for the three-matrix rings (fp32 M3/M4, fp16 M4): parity, sustained A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gather4 or all_variants or full_size or whole" > gpurun_out/r02bp_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r02bp_parity.log
O=gpurun_out/r02bp_gather3.txt
for g in 1 0 1 0; do
  echo "== CD_RING_GATHER=$g" >> $O
  CD_RING_GATHER=$g timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_GATHER=$g timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp32 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_GATHER=$g timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
done
cat $O
