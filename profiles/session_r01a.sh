#!/bin/bash
# Round-1 measurement session: variant sweeps, ncu launch list of the bench, ncu full captures.
set -x
O=gpurun_out
S="python profiles/run_apply.py --sweep --json $O/sweep.jsonl"
$S --dims 2 2 2 2 --nvec 24 --prec fp32
$S --dims 4 4 4 4 --nvec 24 --prec fp32
$S --dims 4 4 4 4 --nvec 24 --prec fp16
$S --dims 8 8 8 8 --nvec 24 --prec fp32
$S --dims 8 8 8 8 --nvec 24 --prec fp32 --cold
$S --dims 8 8 8 8 --nvec 24 --prec fp16
$S --dims 6 6 6 12 --nvec 32 --prec fp32
$S --dims 16 16 16 32 --nvec 24 --prec fp16
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu > $O/bench_under_ncu.log 2>&1
for v in 0 4; do
  ncu --set full --clock-control none --import-source on -k regex:dslash -s 3 -c 1 -f -o $O/prof_8444_f32_v$v \
      python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant $v --reps 5 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:dslash -s 3 -c 1 -f -o $O/prof_8444_f16_v0 \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variant 0 --reps 5 > /dev/null 2>&1
ls -la $O
