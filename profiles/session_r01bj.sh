#!/bin/bash
# Round-1 session bj: what the chain variants do at 4^4 (M2, latency regime) vs single applies in a graph.
O=gpurun_out
for p in fp32 fp16; do
timeout 600 python profiles/run_chain_sweep.py --dims 4 4 4 4 --nvec 24 --prec $p --n 400 >> $O/bj_chain.jsonl 2>> $O/bj.err
timeout 600 python profiles/run_apply.py --dims 4 4 4 4 --nvec 24 --prec $p --sweep --graph --reps 200 >> $O/bj_graph.txt 2>> $O/bj.err
done
cut -c1-200 $O/bj_chain.jsonl; tail -40 $O/bj_graph.txt; tail -3 $O/bj.err
