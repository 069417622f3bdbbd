#!/bin/bash
# round 2, session aj: multi-RHS producer L2 prefetch A/B (CD_MRHS_PF: 1 = next item's links,
# 2 = its neighbour blocks, 3 = both; CD_MRHS_PFD = items ahead); 8^4 x 128 nv24 and M4 x 128 nv32
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
 for cfg in "0 1" "1 1" "1 2" "2 1" "3 1" "3 2"; do
  set -- $cfg
  for d in "8 8 8 8 24" "6 6 6 12 32" "8 8 8 16 24"; do
   set -- $cfg $d
   CD_MRHS_PF=$1 CD_MRHS_PFD=$2 CD_LIB_PATH=ab_libs/mrhs_pf.so timeout 300 python profiles/run_mrhs.py --dims $3 $4 $5 $6 --nvec $7 --nrhs 128 --reps 20 2>&1 | tail -1 | cut -c1-110 | sed "s/^/pf=$1 pfd=$2 /" >> gpurun_out/r02aj_mrhs_pf.txt
  done
 done
done
CD_MRHS_PF=3 CD_LIB_PATH=ab_libs/mrhs_pf.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02aj_parity.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/r02aj_parity.log
cat gpurun_out/r02aj_mrhs_pf.txt
# what bounds the 4^4 per-call apply: ncu --set full of fg_kw3_wr4 (fp32) in a chain of applies
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_fg -s 5 -c 1 -o gpurun_out/r02aj_m2_fg_prof \
  python profiles/run_apply.py --dims 4 4 4 4 --nvec 24 --prec fp32 --variant 5 --reps 8 > gpurun_out/r02aj_m2_ncu.log 2>&1
echo "ncu rc=$?"; head -3 gpurun_out/r02aj_m2_ncu.log
