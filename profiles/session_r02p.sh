#!/bin/bash
# round 2, session p: fused split with the pack on the producer warp's idle lanes (lanes) vs the
# all-CTA prologue (prologue), sustained; launch lists; parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for lib in prologue lanes prologue lanes; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 600 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 1 | sed "s/^/$lib T /" >> gpurun_out/r02p_split.txt
  CD_LIB_PATH=ab_libs/$lib.so timeout 600 python profiles/split_sustained.py --mask 12 --secs 1.0 --rounds 1 | sed "s/^/$lib ZT /" >> gpurun_out/r02p_split.txt
done
CD_LIB_PATH=ab_libs/lanes.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02p_split_lanes.csv \
  python profiles/run_split.py --mask 8 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_self or fused" > gpurun_out/r02p_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -k "peer" > gpurun_out/r02p_multirank.log 2>&1
echo "multirank rc=$?"
cat gpurun_out/r02p_split.txt
