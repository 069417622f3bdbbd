#!/bin/bash
# round 2, session bi: multi-RHS merged hand-offs (exp 64: bfull alone gates the MMA, one commit per hop)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CD_MRHS_EXP=96 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02bi_parity.log 2>&1
echo "parity(96) rc=$?"; tail -2 gpurun_out/r02bi_parity.log
O=gpurun_out/r02bi_merged.txt
for d in "8 8 8 8 24" "6 6 6 12 32"; do
 set -- $d
 for e in 32 96 32 96 64; do
  echo "exp=$e $(CD_MRHS_EXP=$e timeout 120 python profiles/run_mrhs.py --dims $1 $2 $3 $4 --nvec $5)" >> $O
 done
done
for e in 96; do
  CD_MRHS_EXP=$e CD_MRHS_TRACE=gpurun_out/r02bi_tr_$e.bin timeout 120 python profiles/run_mrhs.py --reps 1 > /dev/null 2>&1
  echo "== exp=$e" >> $O
  python profiles/mrhs_trace.py gpurun_out/r02bi_tr_$e.bin 3 5 >> $O 2>&1
done
cat $O
