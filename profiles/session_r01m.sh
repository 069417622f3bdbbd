#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "chain" 2>&1 | tail -2
S="python profiles/run_apply.py --sweep --json $O/sweep_m.jsonl"
$S --dims 2 2 2 2 --nvec 24 --prec fp32 --chain
$S --dims 2 2 2 2 --nvec 24 --prec fp16 --chain
