#!/bin/bash
# Round-1 session ag: barrier-free cluster push chain (variant 4000) -- parity, sanitizers, timing, trace.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain" > $O/ag_pytest.log 2>&1; echo "pytest rc $?" >> $O/ag_pytest.log
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 > $O/ag_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/ag_san_$tool.log
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 3 1 5 1 >> $O/ag_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/ag_san_$tool.log
done
for d in "2 1 1 1" "2 2 2 2"; do
timeout 300 python profiles/run_chain_sweep.py --dims $d --nvec 24 --n 2000 --variants 4000 3002 >> $O/ag_sweep.jsonl 2>> $O/ag_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/ag_trace.bin --trace-variant 4000 >> $O/ag_sweep.jsonl 2>> $O/ag_sweep.err
tail -5 $O/ag_pytest.log; tail -3 $O/ag_san_*.log; cat $O/ag_sweep.jsonl; tail -5 $O/ag_sweep.err; python profiles/cpush_trace.py $O/ag_trace.bin
