#!/bin/bash
# round 2, session e: A/B of the ring consumer's straight-line (no per-hop branch) stage under
# sustained load, alternating old / new library processes; then the gpu parity subset for rings
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
 for lib in old new; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 9 10 --secs 1.0 --rounds 1 | sed "s/^/$lib M5 /" >> gpurun_out/r02e_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 9 10 --secs 0.7 --rounds 1 | sed "s/^/$lib M3h /" >> gpurun_out/r02e_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M3 /" >> gpurun_out/r02e_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M4h /" >> gpurun_out/r02e_ab.txt
 done
done
CD_LIB_PATH=ab_libs/new.so timeout 300 python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --sweep > gpurun_out/r02e_sweep_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "all_variants or dagger or halo_self or full_size" > gpurun_out/r02e_parity.log 2>&1
echo "parity rc=$?"
cat gpurun_out/r02e_ab.txt | cut -c1-160
