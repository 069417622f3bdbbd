#!/bin/bash
# Round-1 session bn: cluster push chain prologue (link loads, cluster barrier, first applies) from the trace.
O=gpurun_out
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 800 --variants 4000 --trace $O/bn_trace.bin --trace-variant 4000 > $O/bn_sweep.jsonl 2> $O/bn.err
python profiles/cpush_trace.py $O/bn_trace.bin | tail -3
