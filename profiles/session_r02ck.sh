#!/bin/bash
# round 2, session ck: multi-RHS with two CTAs per SM (two independent pipelines): parity + A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02ck_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/r02ck_parity.log
O=gpurun_out/r02ck_2cta.txt
for rep in 1 2; do
for d in "8 8 8 8 24 128" "8 8 8 16 24 128" "4 4 4 4 24 1024"; do
 set -- $d
 for c in 1 0; do
  echo "2cta=$c $(CD_MRHS_2CTA=$c timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5 --nrhs $6)" >> $O
 done
done
done
cat $O
