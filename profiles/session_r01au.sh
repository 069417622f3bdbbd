#!/bin/bash
# Round-1 session au: cluster push chain with X links in shared memory + software-pipelined remote hops.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or tuner" > $O/au_pytest.log 2>&1; echo "pytest rc $?" >> $O/au_pytest.log
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 > $O/au_sweep.jsonl 2> $O/au_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/au_trace.bin --trace-variant 4000 >> $O/au_sweep.jsonl 2>> $O/au_sweep.err
tail -2 $O/au_pytest.log; cat $O/au_sweep.jsonl; python profiles/cpush_trace.py $O/au_trace.bin > $O/au_trace.txt; head -7 $O/au_trace.txt
