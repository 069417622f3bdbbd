#!/bin/bash
# Round-1 session w: LL-register chain -- parity tests, sanitizers, tuned sweep, bench line.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain" > $O/w_pytest.log 2>&1; echo "rc=$?" >> $O/w_pytest.log
timeout 900 python -m pytest tests/test_sanitizers.py -q -x -k "chain" >> $O/w_pytest.log 2>&1; echo "rc=$?" >> $O/w_pytest.log
: > $O/w_sweep.jsonl
for dims in "2 2 2 2" "3 2 2 2" "2 2 2 1"; do
timeout 300 python profiles/run_chain_sweep.py --dims $dims --nvec 24 >> $O/w_sweep.jsonl 2>> $O/w_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 32 >> $O/w_sweep.jsonl 2>> $O/w_sweep.err
timeout 600 python bench.py > $O/w_bench.json 2> $O/w_bench.err
tail -4 $O/w_pytest.log; cat $O/w_bench.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['also']['2^4_fp32_chain'], d['value'])"
