#!/bin/bash
# round 2, session bf: multi-RHS CTA-0 event traces: default (link first), no copies (exp 12|32), no build (exp 1|32)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02bg_traces.txt
for e in 32 34 46; do
  CD_MRHS_EXP=$e CD_MRHS_TRACE=gpurun_out/r02bg_tr_$e.bin timeout 120 python profiles/run_mrhs.py --reps 1 > /dev/null 2>&1
  echo "== exp=$e" >> $O
  python profiles/mrhs_trace.py gpurun_out/r02bg_tr_$e.bin 3 5 >> $O 2>&1
done
cat $O
