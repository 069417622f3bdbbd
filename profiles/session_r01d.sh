#!/bin/bash
# Round-1 session d: full ring + prefetch prologue; fp16 row-split fg variants.
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
S="python profiles/run_apply.py --sweep --json $O/sweep_d.jsonl"
$S --dims 8 8 8 8 --nvec 24 --prec fp32 --graph
$S --dims 8 8 8 8 --nvec 24 --prec fp16 --graph
$S --dims 6 6 6 12 --nvec 32 --prec fp32 --graph
$S --dims 16 16 16 32 --nvec 24 --prec fp16
$S --dims 4 4 4 4 --nvec 24 --prec fp16 --graph
$S --dims 2 2 2 2 --nvec 24 --prec fp16 --graph
