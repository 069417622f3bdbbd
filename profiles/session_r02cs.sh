#!/bin/bash
# round 2, session cs: final verification -- smoke, full GPU suite, bench with its tune cache, launch list of the same
# command, ncu --set full of the multi-RHS kernel, reference arm, 2-rank same-GPU bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02cs_smoke.log 2>&1
echo "smoke rc=$?"
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02cs_gpu_suite.log 2>&1
echo "gpu suite rc=$?"; tail -1 gpurun_out/r02cs_gpu_suite.log
export CD_TUNE_CACHE=gpurun_out/r02cs_tune_cache.txt
t0=$(date +%s)
timeout 900 python bench.py > gpurun_out/r02cs_bench.json 2> gpurun_out/r02cs_bench.err
echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02cs_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/r02cs_bench_under_ncu.json 2>&1
echo "launch list rc=$?"
unset CD_TUNE_CACHE
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_mrhs -s 1 -c 1 -o gpurun_out/r02cs_mrhs_prof \
  python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 128 --reps 2 > gpurun_out/r02cs_mrhs_ncu.log 2>&1
echo "mrhs ncu rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02cs_ref.json 2> gpurun_out/r02cs_ref.err
echo "reference arm rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 2 --steps 10 --warmup 3 --same-gpu > gpurun_out/r02cs_bench_2rank.json 2> gpurun_out/r02cs_bench_2rank.err
echo "2-rank bench rc=$?"
tail -3 gpurun_out/r02cs_smoke.log
