#!/bin/bash
# Round-1 session av: cluster push chain with row-group x chunk layout (one shared load per hop), reduce-scatter shuffles, triple reduction.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or tuner" > $O/av_pytest.log 2>&1; echo "pytest rc $?" >> $O/av_pytest.log
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 > $O/av_sweep.jsonl 2> $O/av_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/av_trace.bin --trace-variant 4000 >> $O/av_sweep.jsonl 2>> $O/av_sweep.err
tail -2 $O/av_pytest.log; cat $O/av_sweep.jsonl; python profiles/cpush_trace.py $O/av_trace.bin > $O/av_trace.txt; head -7 $O/av_trace.txt
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 4000 > $O/av_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/av_san_$tool.log
done
grep -h "rc \|SUMMARY" $O/av_san_*.log
