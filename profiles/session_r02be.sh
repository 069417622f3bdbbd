#!/bin/bash
# round 2, session be: multi-RHS SS (link-first default) vs TS with 5/4 A slots in TMEM
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02be_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/r02be_parity.log
O=gpurun_out/r02be_ts_ab.txt
for rep in 1 2; do
for d in "8 8 8 8 24 128" "6 6 6 12 32 128" "8 8 8 16 24 128"; do
 set -- $d
 for ts in 1 0; do
  echo "ts=$ts $(CD_MRHS_TS=$ts timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5 --nrhs $6)" >> $O
 done
done
done
cat $O
