#!/bin/bash
# Round-1 session ac: cluster push chain (variant 4000) -- parity tests, then the 2^4 sweep vs the LL-register chain.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain_tuner" > $O/ac_pytest.log 2>&1; echo "pytest rc $?" >> $O/ac_pytest.log
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 1000 > $O/ac_sweep.jsonl 2> $O/ac_sweep.err
tail -15 $O/ac_pytest.log; cat $O/ac_sweep.jsonl; tail -5 $O/ac_sweep.err
