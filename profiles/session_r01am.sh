#!/bin/bash
# Round-1 session am: LL-warp chain (variant 5000) -- parity, sanitizers, 2^4 timing vs the LL-register chain.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "chain" > $O/am_pytest.log 2>&1; echo "pytest rc $?" >> $O/am_pytest.log
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 5000 > $O/am_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/am_san_$tool.log
done
for d in "2 2 2 2" "2 1 1 1" "3 3 3 3"; do
timeout 300 python profiles/run_chain_sweep.py --dims $d --nvec 24 --n 2000 --variants 5000 3002 >> $O/am_sweep.jsonl 2>> $O/am_sweep.err
done
for d0 in 0 150 450; do
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 5000 --d0 $d0 >> $O/am_sweep.jsonl 2>> $O/am_sweep.err
done
tail -3 $O/am_pytest.log; grep -h "rc \|SUMMARY" $O/am_san_*.log; cat $O/am_sweep.jsonl; tail -5 $O/am_sweep.err
