#!/bin/bash
# round 2, session bd: multi-RHS: per-warp link release (exp 16), link on its own barrier issued first (exp 32)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bd_mrhs_release.txt
for d in "8 8 8 8 24" "6 6 6 12 32"; do
 set -- $d
 for e in 0 16 32 48 0 16 32 48 15 31; do
  echo "exp=$e $(CD_MRHS_EXP=$e timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5)" >> $O
 done
done
cat $O
CD_MRHS_EXP=48 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs_tensor" > gpurun_out/r02bd_parity.log 2>&1
echo "parity(48) rc=$?"; tail -2 gpurun_out/r02bd_parity.log
