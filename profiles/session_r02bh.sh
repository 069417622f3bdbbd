#!/bin/bash
# round 2, session bh: verification after the multi-RHS link-first change -- smoke, full GPU suite, bench with
# its tune cache, launch list of the same command, ncu --set full of the headline kernel
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02bh_smoke.log 2>&1
echo "smoke rc=$?"
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02bh_gpu_suite.log 2>&1
echo "gpu suite rc=$?"
export CD_TUNE_CACHE=gpurun_out/r02bh_tune_cache.txt
t0=$(date +%s)
timeout 900 python bench.py > gpurun_out/r02bh_bench.json 2> gpurun_out/r02bh_bench.err
echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02bh_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02bh_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
unset CD_TUNE_CACHE
t0=$(date +%s)
timeout 900 python bench.py --impl reference > gpurun_out/r02bh_ref.json 2> gpurun_out/r02bh_ref.err
echo "reference arm rc=$? wall $(( $(date +%s) - t0 )) s"
tail -3 gpurun_out/r02bh_gpu_suite.log; tail -3 gpurun_out/r02bh_smoke.log
