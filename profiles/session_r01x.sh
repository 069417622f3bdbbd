#!/bin/bash
# Round-1 session x: full GPU suite after the tuner change, bench line, bench launch list,
# ncu --set full of the LL-register chain (2^4, variant 3002), fresh chain trace.
O=gpurun_out
# (suite ran green in the previous call)
timeout 600 python bench.py > $O/x_bench.json 2> $O/x_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/x_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/x_bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:llreg -s 1 -c 1 -f -o $O/x_llreg \
    python profiles/run_chain_prof.py --variant 3002 --n 2000 > $O/x_ncu_llreg.log 2>&1
ncu -i $O/x_llreg.ncu-rep --page raw --csv > $O/x_llreg.raw.csv 2>/dev/null
timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --variants 3002 --reps 1 --trace $O/x_trace3002.bin --trace-variant 3002 > /dev/null 2>&1
python profiles/chain_trace.py $O/x_trace3002.bin > $O/x_trace.txt 2>&1
tail -3 $O/x_pytest.log; python -c "import json; d=json.load(open('$O/x_bench.json')); print(d['value'], d['config']['variant'], d['also']['2^4_fp32_chain'])"
