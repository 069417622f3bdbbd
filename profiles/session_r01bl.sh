#!/bin/bash
# Round-1 session bl: 2^4 chain timing with finite data throughout (800 applies per launch, vector re-imported
# before every timed launch) vs the earlier 2000-apply protocol (the iterate overflowed after ~1000 applies).
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "long_chain" > $O/bl_pytest.log 2>&1; echo "pytest rc $?" >> $O/bl_pytest.log
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 4000 3002 > $O/bl_sweep800.jsonl 2>> $O/bl.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 > $O/bl_sweep2000.jsonl 2>> $O/bl.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu > $O/bl_bench.json 2> $O/bl_bench.err
tail -2 $O/bl_pytest.log; cut -c1-175 $O/bl_sweep800.jsonl $O/bl_sweep2000.jsonl
python -c "import json; d=json.load(open('$O/bl_bench.json')); print(d['also'].get('2^4_fp32_chain'))"
