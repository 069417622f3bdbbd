#!/bin/bash
# Round-1 session z: LL-register chain with 256-bit per-chunk polls (no smem staging).
O=gpurun_out
: > $O/z_sweep.jsonl
for d0 in 0 300; do
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 2001 $(seq 3001 3006) --d0 $d0 >> $O/z_sweep.jsonl 2>> $O/z_sweep.err
done
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 32 --variants $(seq 3001 3006) >> $O/z_sweep.jsonl 2>> $O/z_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 3 2 2 2 --nvec 24 --variants $(seq 3001 3006) >> $O/z_sweep.jsonl 2>> $O/z_sweep.err
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 3002 --reps 1 --trace $O/z_trace3002.bin --trace-variant 3002 > /dev/null 2>> $O/z_sweep.err
python profiles/chain_trace.py $O/z_trace3002.bin > $O/z_trace.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "llreg" > $O/z_pytest.log 2>&1; echo "rc=$?" >> $O/z_pytest.log
cat $O/z_trace.txt; tail -3 $O/z_pytest.log; tail -3 $O/z_sweep.err
