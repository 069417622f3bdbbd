#!/bin/bash
O=gpurun_out
for v in 0 2; do
ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/prof_8444_f16_v$v \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variant $v --reps 6 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/prof_8444_f32_ring \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant 0 --reps 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/prof_8444_f32_fg34 \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant 5 --reps 6 > /dev/null 2>&1
ls $O/*.ncu-rep
