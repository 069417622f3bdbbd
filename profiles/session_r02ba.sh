#!/bin/bash
# round 2, session ba: multi-RHS stage-lifetime decomposition (diagnostic knobs: ring depth cap, skip B build / MMA /
# link copy / A copy) at 8^4 x 128 and 6^3x12 x 128
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02ba_mrhs_knobs.txt
for d in "8 8 8 8 24" "6 6 6 12 32"; do
 set -- $d
 for smax in 0 4 3 2; do
  echo "smax=$smax $(CD_MRHS_SMAX=$smax timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5)" >> $O
 done
 for e in 1 2 3 4 8 5 9; do
  echo "exp=$e $(CD_MRHS_EXP=$e timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5)" >> $O
 done
done
CD_MRHS_TRACE=gpurun_out/r02ba_tr.bin timeout 120 python profiles/run_mrhs.py --reps 1 >/dev/null 2>&1
python profiles/mrhs_trace.py gpurun_out/r02ba_tr.bin >> $O 2>&1
cat $O
