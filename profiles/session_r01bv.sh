#!/bin/bash
# Round-1 session bv: cluster push chain with the remote wait no longer forced after the X math -- parity,
# sanitizers, trace, bench.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain" > $O/bv_pytest.log 2>&1; echo "pytest rc $?" >> $O/bv_pytest.log
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 4000 > $O/bv_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bv_san_$tool.log
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 3 1 5 1 4000 >> $O/bv_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bv_san_$tool.log
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 4000 3002 > $O/bv_sweep.jsonl 2>> $O/bv.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 200 --variants 4000 >> $O/bv_sweep.jsonl 2>> $O/bv.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 4000 --trace $O/bv_trace.bin --trace-variant 4000 >> $O/bv_sweep.jsonl 2>> $O/bv.err
timeout 600 python bench.py --no-cpu > $O/bv_bench.json 2> $O/bv_bench.err
tail -2 $O/bv_pytest.log; grep -h "rc \|SUMMARY" $O/bv_san_*.log; cut -c1-175 $O/bv_sweep.jsonl; python profiles/cpush_trace.py $O/bv_trace.bin | head -7
python -c "import json; d=json.load(open('$O/bv_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['also']['2^4_fp32_chain'])"
