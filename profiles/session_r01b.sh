#!/bin/bash
# Round-1 session b: dynamic-ticket ring vs fg; CUDA-graph timing of small lattices.
O=gpurun_out
S="python profiles/run_apply.py --sweep --json $O/sweep_b.jsonl"
$S --dims 2 2 2 2 --nvec 24 --prec fp32 --graph
$S --dims 2 2 2 2 --nvec 24 --prec fp16 --graph
$S --dims 4 4 4 4 --nvec 24 --prec fp32 --graph
$S --dims 4 4 4 4 --nvec 24 --prec fp16 --graph
$S --dims 8 8 8 8 --nvec 24 --prec fp32
$S --dims 8 8 8 8 --nvec 24 --prec fp16
$S --dims 6 6 6 12 --nvec 32 --prec fp32
$S --dims 16 16 16 32 --nvec 24 --prec fp16
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
