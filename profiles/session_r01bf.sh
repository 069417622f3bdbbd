#!/bin/bash
# Round-1 session bf: clock64 trace of the cluster push chain after the early-arrive / sign-fold changes.
O=gpurun_out
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/bf_trace.bin --trace-variant 4000 > $O/bf_sweep.jsonl 2> $O/bf_sweep.err
python profiles/cpush_trace.py $O/bf_trace.bin > $O/bf_trace.txt; head -7 $O/bf_trace.txt; cut -c1-180 $O/bf_sweep.jsonl
