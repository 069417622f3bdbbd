#!/bin/bash
# round 2, session m: rot3 (fused split: rotated order, hoisted fp16 scales, faster pack, unrolled
# producer) vs nopipe (the first fused version): unsplit sustained A/B, split launch lists, parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
 for lib in nopipe rot3; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 9 --secs 1.0 --rounds 1 | sed "s/^/$lib M5 /" >> gpurun_out/r02m_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 0 --secs 0.7 --rounds 1 | sed "s/^/$lib M3 /" >> gpurun_out/r02m_ab.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.7 --rounds 1 | sed "s/^/$lib M4h /" >> gpurun_out/r02m_ab.txt
 done
done
for m in 8 12; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_split_$m.csv \
  python profiles/run_split.py --mask $m --transport peer --variant 10 --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_split_unfused_$m.csv \
  env CD_FUSE_SPLIT=0 python profiles/run_split.py --mask $m --transport peer --variant 10 --reps 3 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_split_m3f32.csv \
  python profiles/run_split.py --dims 8 8 8 8 --prec fp32 --mask 8 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "all_variants or halo_self or full_size" > gpurun_out/r02m_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -k "peer" > gpurun_out/r02m_multirank.log 2>&1
echo "multirank rc=$?"
cut -c1-150 gpurun_out/r02m_ab.txt
