#!/bin/bash
# Round-1 session bk: LL-triple chain (variant 6000) -- parity, sanitizers, timing at 2^4 / 3^4 / 4^4.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "lltri or chain_tuner" > $O/bk_pytest.log 2>&1; echo "pytest rc $?" >> $O/bk_pytest.log
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 6000 > $O/bk_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bk_san_$tool.log
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 3 3 3 3 6000 >> $O/bk_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bk_san_$tool.log
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 6000 4000 3002 >> $O/bk_sweep.jsonl 2>> $O/bk.err
timeout 300 python profiles/run_chain_sweep.py --dims 3 3 3 3 --nvec 24 --n 1000 --variants 6000 5000 >> $O/bk_sweep.jsonl 2>> $O/bk.err
timeout 300 python profiles/run_chain_sweep.py --dims 4 4 4 4 --nvec 24 --n 400 --variants 6000 >> $O/bk_sweep.jsonl 2>> $O/bk.err
timeout 300 python profiles/run_chain_sweep.py --dims 4 4 4 4 --nvec 24 --prec fp16 --n 400 --variants 2002 >> $O/bk_sweep.jsonl 2>> $O/bk.err
tail -2 $O/bk_pytest.log; grep -h "rc \|SUMMARY" $O/bk_san_*.log; cut -c1-190 $O/bk_sweep.jsonl; tail -3 $O/bk.err
