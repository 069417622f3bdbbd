#!/bin/bash
# round 2, session h: bench; ncu --set full of the M5 headline kernel (straight-line ring m9);
# ncu launch list of the bench command
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_ring -s 1 -c 1 -o gpurun_out/r02h_m5_prof \
  python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variant 10 --reps 3 > gpurun_out/r02h_m5_ncu.log 2>&1
echo "m5 ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02h_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
