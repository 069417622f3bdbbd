#!/bin/bash
# round 2, session k: producer ticket/site software pipeline (pipe) vs not (nopipe): unsplit
# sustained A/B on M5 fp16 / M3 fp32 / M4 fp16, split launch lists, parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
 for lib in nopipe pipe; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 9 --secs 1.0 --rounds 1 | sed "s/^/$lib M5 /" >> gpurun_out/r02k_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M3 /" >> gpurun_out/r02k_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.7 --rounds 1 | sed "s/^/$lib M4h /" >> gpurun_out/r02k_ab.txt
 done
done
for lib in nopipe pipe; do
CD_LIB_PATH=ab_libs/$lib.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k_split_$lib.csv \
  python profiles/run_split.py --mask 8 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
CD_LIB_PATH=ab_libs/$lib.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k_nosplit_$lib.csv \
  python profiles/run_split.py --mask 0 --variant 10 --reps 3 > /dev/null 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "all_variants or halo_self or full_size" > gpurun_out/r02k_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -k "operator and peer" > gpurun_out/r02k_multirank.log 2>&1
echo "multirank rc=$?"
cut -c1-150 gpurun_out/r02k_ab.txt
