#!/bin/bash
# round 2, session d: multi-rank parity (peer), sustained-load variant ranking (M5 / M3 fp16, M3 fp32),
# bench with the fixed per-config protocol, the full single-GPU parity suite
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -s -k "operator and peer" > gpurun_out/r02d_multirank.log 2>&1
echo "multirank rc=$?"
timeout 600 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 9 10 0 1 2 --secs 0.5 --rounds 3 --json gpurun_out/r02d_sustained.jsonl > gpurun_out/r02d_sustained_m5.txt 2>&1
timeout 600 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 9 10 0 1 2 --secs 0.5 --rounds 3 --json gpurun_out/r02d_sustained.jsonl > gpurun_out/r02d_sustained_m3h.txt 2>&1
timeout 600 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variants 10 0 5 4 --secs 0.5 --rounds 3 --json gpurun_out/r02d_sustained.jsonl > gpurun_out/r02d_sustained_m3.txt 2>&1
echo "sustained done"
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
echo "bench rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02d_parity.log 2>&1
echo "parity rc=$?"
tail -3 gpurun_out/r02d_multirank.log gpurun_out/r02d_parity.log
