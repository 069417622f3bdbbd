#!/bin/bash
# Round-1 session bm: chain timing without host submission latency in the event window (spin kernel ahead of
# the start event) and with the cluster-occupancy query cached; 800 and 2000 applies per launch.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cpush or long_chain or chain_tuner" > $O/bm_pytest.log 2>&1; echo "pytest rc $?" >> $O/bm_pytest.log
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 4000 3002 > $O/bm_sweep800.jsonl 2>> $O/bm.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 200 --variants 4000 3002 > $O/bm_sweep200.jsonl 2>> $O/bm.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 > $O/bm_sweep2000.jsonl 2>> $O/bm.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu > $O/bm_bench.json 2> $O/bm_bench.err
tail -2 $O/bm_pytest.log; cut -c1-175 $O/bm_sweep800.jsonl $O/bm_sweep200.jsonl $O/bm_sweep2000.jsonl
python -c "import json; d=json.load(open('$O/bm_bench.json')); print(d['also'].get('2^4_fp32_chain'))"
