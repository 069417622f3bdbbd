#!/bin/bash
# round 2, session bl: ring m9 with two consumer groups (variant 11, ring_tma_m9g2_f16_nv24): parity, sustained A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02bl_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/r02bl_parity.log
O=gpurun_out/r02bl_g2.txt
timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 11 --secs 0.6 --rounds 4 >> $O 2>&1
timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 11 --secs 0.4 --rounds 3 >> $O 2>&1
cat $O
