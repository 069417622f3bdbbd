#!/bin/bash
# round 2, session j: the fused split apply (ring + peer): self-exchange parity, multi-rank parity,
# launch list of split applies, overlap figures
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_self" > gpurun_out/r02j_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -s -k "peer" > gpurun_out/r02j_multirank.log 2>&1
echo "multirank rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_split_peer.csv \
  python profiles/run_split.py --mask 8 --transport peer --variant 10 --reps 4 > gpurun_out/r02j_split_peer.log 2>&1
echo "launch list rc=$?"
timeout 900 python bench.py --no-cpu > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
echo "bench rc=$?"
tail -3 gpurun_out/r02j_parity.log; tail -3 gpurun_out/r02j_multirank.log
