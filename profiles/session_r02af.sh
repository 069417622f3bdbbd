#!/bin/bash
# round 2, session af: verification after the kernel changes -- smoke, full GPU suite, bench with
# its tune cache, launch list of the same command, ncu --set full of the headline kernel
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02af_smoke.log 2>&1
echo "smoke rc=$?"
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02af_gpu_suite.log 2>&1
echo "gpu suite rc=$?"
export CD_TUNE_CACHE=gpurun_out/r02af_tune_cache.txt
timeout 900 python bench.py > gpurun_out/r02af_bench.json 2> gpurun_out/r02af_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02af_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02af_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
unset CD_TUNE_CACHE
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_ring -s 1 -c 1 -o gpurun_out/r02af_m5_prof \
  python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variant 10 --reps 3 > gpurun_out/r02af_m5_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02af_gpu_suite.log; tail -3 gpurun_out/r02af_smoke.log
