#!/bin/bash
# round 2, session ai: verification after the fg direct-load change -- smoke, full GPU suite, bench with
# its tune cache, launch list of the same command, ncu --set full of the headline kernel
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02ai_smoke.log 2>&1
echo "smoke rc=$?"
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02ai_gpu_suite.log 2>&1
echo "gpu suite rc=$?"
export CD_TUNE_CACHE=gpurun_out/r02ai_tune_cache.txt
timeout 900 python bench.py > gpurun_out/r02ai_bench.json 2> gpurun_out/r02ai_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ai_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02ai_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
unset CD_TUNE_CACHE
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_ring -s 1 -c 1 -o gpurun_out/r02ai_m5_prof \
  python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variant 10 --reps 3 > gpurun_out/r02ai_m5_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02ai_gpu_suite.log; tail -3 gpurun_out/r02ai_smoke.log
# the gated direct loads vs the staged path (profiles/r02/fg_direct_ab.txt had the ungated A/B)
for lib in nodirect direct2; do
 for d in "2 2 2 2" "4 4 4 4"; do
  for p in fp32 fp16; do
   CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/run_apply.py --dims $d --nvec 24 --prec $p --sweep --graph 2>&1 | grep fg_kw1 | sed "s/^/$lib /" >> gpurun_out/r02ai_direct_gated.txt
  done
 done
done
