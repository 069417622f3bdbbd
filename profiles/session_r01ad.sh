#!/bin/bash
# Round-1 session ad: cluster push chain timing on 1^4 / 2x1x1x1 / 2^4 and a clock64 trace at 2^4.
O=gpurun_out
for d in "1 1 1 1" "2 1 1 1" "2 2 1 1" "2 2 2 2"; do
timeout 300 python profiles/run_chain_sweep.py --dims $d --nvec 24 --n 2000 --variants 4000 >> $O/ad_sweep.jsonl 2>> $O/ad_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/ad_trace.bin --trace-variant 4000 >> $O/ad_sweep.jsonl 2>> $O/ad_sweep.err
cat $O/ad_sweep.jsonl; tail -5 $O/ad_sweep.err; python profiles/cpush_trace.py $O/ad_trace.bin
