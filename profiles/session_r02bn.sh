#!/bin/bash
# round 2, session bn: ring m9 producer with TMA gather4 for the neighbour vector records: parity + sustained A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02bn_parity.log 2>&1
echo "parity rc=$?"; tail -4 gpurun_out/r02bn_parity.log
O=gpurun_out/r02bn_gather.txt
for g in 1 0 1 0; do
  echo "== CD_RING_GATHER=$g" >> $O
  CD_RING_GATHER=$g timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 3 >> $O 2>&1
  CD_RING_GATHER=$g timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
done
cat $O
