#!/bin/bash
# Round-1 session ak: cluster push chain (variant 4000) with FFMA2 math -- parity, timing, trace.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain" > $O/ak_pytest.log 2>&1; echo "pytest rc $?" >> $O/ak_pytest.log
for d in "2 1 1 1" "2 2 2 2"; do
timeout 300 python profiles/run_chain_sweep.py --dims $d --nvec 24 --n 2000 --variants 4000 3002 >> $O/ak_sweep.jsonl 2>> $O/ak_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/ak_trace.bin --trace-variant 4000 >> $O/ak_sweep.jsonl 2>> $O/ak_sweep.err
tail -3 $O/ak_pytest.log; cat $O/ak_sweep.jsonl; tail -5 $O/ak_sweep.err; python profiles/cpush_trace.py $O/ak_trace.bin | head -14
timeout 600 compute-sanitizer --tool racecheck --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 > $O/ak_san.log 2>&1; echo "racecheck rc $?" >> $O/ak_san.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode=3 python profiles/cpush_debug.py 3 1 5 1 >> $O/ak_san.log 2>&1; echo "synccheck rc $?" >> $O/ak_san.log
grep "rc \|SUMMARY" $O/ak_san.log
