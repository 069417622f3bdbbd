#!/bin/bash
# Round-1 session ai: cluster push chain (variant 4000) with FFMA2 math -- parity, timing, trace.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain" > $O/ai_pytest.log 2>&1; echo "pytest rc $?" >> $O/ai_pytest.log
for d in "2 1 1 1" "2 2 2 2"; do
timeout 300 python profiles/run_chain_sweep.py --dims $d --nvec 24 --n 2000 --variants 4000 3002 >> $O/ai_sweep.jsonl 2>> $O/ai_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 --trace $O/ai_trace.bin --trace-variant 4000 >> $O/ai_sweep.jsonl 2>> $O/ai_sweep.err
tail -3 $O/ai_pytest.log; cat $O/ai_sweep.jsonl; tail -5 $O/ai_sweep.err; python profiles/cpush_trace.py $O/ai_trace.bin | head -14
