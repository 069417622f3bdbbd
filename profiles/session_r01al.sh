#!/bin/bash
# Round-1 session al: cluster push chain trace with the waits skipped (math + epilogue alone).
O=gpurun_out
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --d1 -1 --trace $O/al_trace.bin --trace-variant 4000 > $O/al_sweep.jsonl 2> $O/al_sweep.err
python profiles/cpush_trace.py $O/al_trace.bin > $O/al_trace.txt; head -7 $O/al_trace.txt; tail -3 $O/al_sweep.err
