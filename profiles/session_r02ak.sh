#!/bin/bash
# round 2, session ak: multi-RHS B builders loading the link records from global memory one hop
# ahead (CD_MRHS_LG=1; ring stage = neighbour block only) vs the ring-staged links; with/without
# the one-item-ahead L2 prefetch of the links (CD_MRHS_PF=1); B-slot count (CD_MRHS_NBS)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
 for cfg in "0 0 0" "0 1 0" "1 0 0" "1 1 0" "1 1 9"; do
  for d in "8 8 8 8 24" "6 6 6 12 32" "8 8 8 16 24"; do
   set -- $cfg $d
   CD_MRHS_LG=$1 CD_MRHS_PF=$2 CD_MRHS_NBS=$3 CD_LIB_PATH=ab_libs/mrhs_lg.so timeout 300 python profiles/run_mrhs.py --dims $4 $5 $6 $7 --nvec $8 --nrhs 128 --reps 20 2>&1 | tail -1 | cut -c1-110 | sed "s/^/lg=$1 pf=$2 nbs=$3 /" >> gpurun_out/r02ak_mrhs_lg.txt
  done
 done
done
for lg in 0 1; do
CD_MRHS_LG=$lg CD_MRHS_PF=1 CD_LIB_PATH=ab_libs/mrhs_lg.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02ak_parity_lg$lg.log 2>&1
echo "parity lg=$lg rc=$?"; tail -1 gpurun_out/r02ak_parity_lg$lg.log
done
CD_MRHS_LG=1 CD_MRHS_PF=1 CD_LIB_PATH=ab_libs/mrhs_lg.so timeout 600 python -m pytest tests/test_sanitizers.py -q -x -k "mrhs" > gpurun_out/r02ak_san.log 2>&1
echo "sanitizers rc=$?"; tail -1 gpurun_out/r02ak_san.log
cat gpurun_out/r02ak_mrhs_lg.txt
