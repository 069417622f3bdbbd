#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
S="python profiles/run_apply.py --sweep --json $O/sweep_g.jsonl"
$S --dims 8 8 8 8 --nvec 24 --prec fp32 --graph
$S --dims 8 8 8 8 --nvec 24 --prec fp16 --graph
$S --dims 16 16 16 32 --nvec 24 --prec fp16
$S --dims 6 6 6 12 --nvec 32 --prec fp32 --graph
