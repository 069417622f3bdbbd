#!/bin/bash
# Round-1 session ae: barrier-free cluster push chain (variant 4000) -- parity, timing, trace.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain_tuner" > $O/ae_pytest.log 2>&1; echo "pytest rc $?" >> $O/ae_pytest.log
for d in "1 1 1 1" "2 2 2 2"; do
timeout 300 python profiles/run_chain_sweep.py --dims $d --nvec 24 --n 2000 --variants 4000 3002 >> $O/ae_sweep.jsonl 2>> $O/ae_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/ae_trace.bin --trace-variant 4000 >> $O/ae_sweep.jsonl 2>> $O/ae_sweep.err
tail -15 $O/ae_pytest.log; cat $O/ae_sweep.jsonl; tail -5 $O/ae_sweep.err; python profiles/cpush_trace.py $O/ae_trace.bin
