#!/bin/bash
# round 2, session l: fused split apply with rotated (arithmetic) ticket order: launch lists,
# self-halo overlap in the bench, parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_split_rot.csv \
  python profiles/run_split.py --mask 8 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_split_zt.csv \
  python profiles/run_split.py --mask 12 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_nosplit.csv \
  python profiles/run_split.py --mask 0 --variant 10 --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_split_unfused.csv \
  env CD_FUSE_SPLIT=0 python profiles/run_split.py --mask 8 --transport peer --variant 10 --reps 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_self" > gpurun_out/r02l_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -k "peer" > gpurun_out/r02l_multirank.log 2>&1
echo "multirank rc=$?"
timeout 900 python bench.py --no-cpu > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err
echo "bench rc=$?"
