#!/bin/bash
# ncu --set full of the top 8^4 variants (fp32: fg kw3 wr2/wr4/wr6, ring m1; fp16: ring m9/m3, fg kw9 wr6),
# the LL chain at 2^4 and the tcgen05 multi-RHS kernel -> traffic per launch for bench.py.
O=gpurun_out
for v in 4 5 6 0; do
  ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/r01q_f32_v$v \
      python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant $v --reps 6 > /dev/null 2>&1
done
for v in 10 9 2; do
  ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/r01q_f16_v$v \
      python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variant $v --reps 6 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:mrhs -s 3 -c 1 -f -o $O/r01q_mrhs \
    python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 128 --reps 2 > /dev/null 2>&1
ls $O/r01q_*
