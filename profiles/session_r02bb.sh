#!/bin/bash
# round 2, session bb: multi-RHS TS variant (links as the A operand in tensor memory): parity, racecheck, A/B timing
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02bb_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r02bb_parity.log
O=gpurun_out/r02bb_ts_ab.txt
for rep in 1 2; do
for d in "8 8 8 8 24 128" "6 6 6 12 32 128" "4 4 4 4 24 1024" "8 8 8 16 24 128"; do
 set -- $d
 for ts in 1 0; do
  echo "ts=$ts $(CD_MRHS_TS=$ts timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5 --nrhs $6)" >> $O
 done
done
done
cat $O
timeout 900 python -m pytest tests/test_sanitizers.py -q -x -k "mrhs" > gpurun_out/r02bb_san.log 2>&1
echo "san rc=$?"; tail -3 gpurun_out/r02bb_san.log
