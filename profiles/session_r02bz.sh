#!/bin/bash
# round 2, session bz: fp16 ring with deferred quantisation (no per-site cross-warp barrier): parity + same-box A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r02bz_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r02bz_parity.log
O=gpurun_out/r02bz_dq.txt
for e in 0 8 0 8; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
done
cat $O
