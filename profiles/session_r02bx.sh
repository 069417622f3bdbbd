#!/bin/bash
# round 2, session bx: fp16 ring with a dedicated epilogue warp (consumers hand rows over, no per-site barrier)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r02bx_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r02bx_parity.log
O=gpurun_out/r02bx_epw.txt
for e in 0 32 0 32; do
  echo "== CD_RING_EXP=$e" >> $O
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 3 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
  CD_RING_EXP=$e timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
done
CD_RING_EXP=2 timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 2 >> $O 2>&1
cat $O
