#!/bin/bash
# round 2, session f: A/B whole-site ring consumer (new2) vs per-stage straight-line (new) under
# sustained load; parity of the ring variants; multi-rank bench path on one GPU (--same-gpu);
# full bench with the self-halo overlap measurement
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
 for lib in new new2; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 9 10 0 --secs 1.0 --rounds 1 | sed "s/^/$lib M5 /" >> gpurun_out/r02f_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M3 /" >> gpurun_out/r02f_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M4h /" >> gpurun_out/r02f_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp32 --variants 8 0 1 --secs 0.7 --rounds 1 | sed "s/^/$lib M4 /" >> gpurun_out/r02f_ab.txt
 done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "all_variants or dagger or halo_self or full_size or impulse or shift" > gpurun_out/r02f_parity.log 2>&1
echo "parity rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --same-gpu > gpurun_out/r02f_bench_2rank_samegpu.json 2> gpurun_out/r02f_bench_2rank.err
echo "2-rank bench rc=$?"
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
echo "bench rc=$?"
cut -c1-170 gpurun_out/r02f_ab.txt; tail -2 gpurun_out/r02f_parity.log
