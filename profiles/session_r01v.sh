#!/bin/bash
# Round-1 session v: LL-register chain with paired +mu/-mu polls (L_mu = 2).
O=gpurun_out
: > $O/v_sweep.jsonl
for d0 in 0 200 300 400; do
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 3001 3002 3003 3004 3005 --d0 $d0 >> $O/v_sweep.jsonl 2>> $O/v_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 32 --variants 2002 3001 3002 3003 3004 3005 3006 --d0 300 >> $O/v_sweep.jsonl 2>> $O/v_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 3 2 2 2 --nvec 24 --variants 2001 3001 3002 3003 3004 3005 3006 --d0 300 >> $O/v_sweep.jsonl 2>> $O/v_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 3002 --reps 1 --d0 300 --trace $O/v_trace3002.bin --trace-variant 3002 >> /dev/null 2>> $O/v_sweep.err
python profiles/chain_trace.py $O/v_trace3002.bin > $O/v_trace.txt 2>&1
cat $O/v_trace.txt; tail -5 $O/v_sweep.err
