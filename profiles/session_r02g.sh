#!/bin/bash
# round 2, session g: bench (new tuner, straight-line interior in halo mode), halo/transport
# parity, sanitizers over the transports, ncu --set full of the tcgen05 multi-RHS kernel,
# launch list of the bench command
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo or full_size or link_kinds or split_mismatch" > gpurun_out/r02g_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_sanitizers.py -q -x -k "transport or halo or apply" > gpurun_out/r02g_san.log 2>&1
echo "sanitizers rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_mrhs -s 3 -c 1 -o gpurun_out/r02g_mrhs_prof \
  python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 128 --reps 2 > gpurun_out/r02g_mrhs_ncu.log 2>&1
echo "mrhs ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dslash_ring -s 40 -c 1 -o gpurun_out/r02g_m5_prof \
  python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variant 10 --reps 3 > gpurun_out/r02g_m5_ncu.log 2>&1
echo "m5 ncu rc=$?"
tail -2 gpurun_out/r02g_parity.log gpurun_out/r02g_san.log
