#!/bin/bash
# Round-1 session az: cluster push chain -- immediate barrier ids; trace with the epilogue split.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush" > $O/az_pytest.log 2>&1; echo "pytest rc $?" >> $O/az_pytest.log
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 > $O/az_sweep.jsonl 2> $O/az_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/az_trace.bin --trace-variant 4000 >> $O/az_sweep.jsonl 2>> $O/az_sweep.err
tail -2 $O/az_pytest.log; cut -c1-170 $O/az_sweep.jsonl; python profiles/cpush_trace.py $O/az_trace.bin > $O/az_trace.txt; head -15 $O/az_trace.txt
