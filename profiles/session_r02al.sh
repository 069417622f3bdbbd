#!/bin/bash
# round 2, session al: ring with two consumer groups taking alternate sites (ring_tma_m*_cg2):
# parity of every variant, sanitizers over the ring variants, sustained-load timing vs the
# one-group rings at M5 / M3 / M4
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02al_parity.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/r02al_parity.log
timeout 900 python -m pytest tests/test_sanitizers.py -q -x -k "apply or ring or transport" > gpurun_out/r02al_san.log 2>&1
echo "sanitizers rc=$?"; tail -1 gpurun_out/r02al_san.log
timeout 600 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 11 9 12 0 --secs 0.5 --rounds 3 > gpurun_out/r02al_m5.txt 2>&1
echo "m5 rc=$?"
timeout 600 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 11 9 12 --secs 0.4 --rounds 3 > gpurun_out/r02al_m3f16.txt 2>&1
timeout 600 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 11 0 --secs 0.4 --rounds 3 > gpurun_out/r02al_m3f32.txt 2>&1
timeout 600 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 9 0 --secs 0.4 --rounds 3 > gpurun_out/r02al_m4f16.txt 2>&1
tail -8 gpurun_out/r02al_m5.txt; tail -5 gpurun_out/r02al_m3f16.txt; tail -4 gpurun_out/r02al_m3f32.txt; tail -4 gpurun_out/r02al_m4f16.txt
