#!/bin/bash
# round 2, session c: multi-rank operator parity (peer, R procs on one GPU), the new bench
# (M5 headline + every BASELINE config), M5 variant sweep, launch list, ncu --set full of the
# M5 headline kernel
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -s -k "operator and peer" > gpurun_out/r02c_multirank.log 2>&1
echo "multirank rc=$?"
timeout 900 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
echo "bench rc=$?"
timeout 600 python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --sweep > gpurun_out/r02c_sweep_m5.txt 2>&1
echo "sweep rc=$?"
VAR=$(python - <<'PY'
import json
d = json.load(open("gpurun_out/r02c_bench.json"))
import sys; sys.path.insert(0, ".")
import paper_1612_07873_b200 as cd
ctx = cd.Context((2, 2, 2, 2), 24)
print(ctx.variants("fp16").index(d["config"]["variant"]))
PY
)
echo "headline variant id=$VAR"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02c_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dslash_ -s 2 -c 1 -o gpurun_out/r02c_m5_prof \
  python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variant $VAR --reps 3 > gpurun_out/r02c_ncu.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/r02c_multirank.log
