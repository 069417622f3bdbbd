#!/bin/bash
# round 2, session am: ncu DRAM traffic per launch (cold caches, ncu default cache control) of the
# variants the bench picks for M1, M2 and M4 -- the configs without a committed traffic figure
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum"
run() {  # tag dims nvec prec variant regex
  timeout 600 ncu --metrics $M --clock-control none -k regex:$6 -s 3 -c 1 --csv \
    python profiles/run_apply.py --dims $2 --nvec $3 --prec $4 --variant $5 --reps 6 > gpurun_out/r02am_$1.csv 2>&1
  echo "$1 rc=$?"
}
run m1_f32 "2 2 2 2" 24 fp32 2 dslash_fg
run m2_f32 "4 4 4 4" 24 fp32 5 dslash_fg
run m2_f16 "4 4 4 4" 24 fp16 2 dslash_fg
run m4_f32 "6 6 6 12" 32 fp32 0 dslash_ring
run m4_f16 "6 6 6 12" 32 fp16 8 dslash_ring
grep -h "variant\|dram__bytes\|gpu__time" gpurun_out/r02am_*.csv | cut -c1-200
