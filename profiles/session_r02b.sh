#!/bin/bash
# round 2, session b: transports (copy / 1-rank NCCL / peer) on one GPU, multi-rank parity with
# R processes on one GPU over the peer transport, robustness tests
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "halo_self or link_kinds or split_mismatch or restore_current" > gpurun_out/r02b_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -x -q -s -k "operator and peer" > gpurun_out/r02b_multirank.log 2>&1
echo "multirank rc=$?"
timeout 1800 python -m pytest tests/test_gpu_multirank.py -x -q -s -k "fullsize and peer" > gpurun_out/r02b_fullsize.log 2>&1
echo "fullsize rc=$?"
tail -5 gpurun_out/r02b_parity.log gpurun_out/r02b_multirank.log gpurun_out/r02b_fullsize.log
