#!/bin/bash
# round 2, session q: scale-quad fused split (quad) vs lanes vs prologue: split/unsplit sustained;
# unsplit ring A/B (consumer unroll); graph-timed tuner choice for M1/M2; parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for lib in lanes quad lanes quad; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 600 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 1 | sed "s/^/$lib T /" >> gpurun_out/r02q_split.txt
done
for lib in rot3 quad rot3 quad; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M3 /" >> gpurun_out/r02q_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M4h /" >> gpurun_out/r02q_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 9 --secs 0.7 --rounds 1 | sed "s/^/$lib M3h /" >> gpurun_out/r02q_ab.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_self or fused or all_variants" > gpurun_out/r02q_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -k "peer" > gpurun_out/r02q_multirank.log 2>&1
echo "multirank rc=$?"
timeout 900 python bench.py --no-cpu > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
echo "bench rc=$?"
cat gpurun_out/r02q_split.txt gpurun_out/r02q_ab.txt | cut -c1-140
