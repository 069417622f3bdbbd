#!/bin/bash
# Round-1 session ar: full GPU suite + smoke + bench (tune cache written) + ncu launch list of the same bench command.
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/ar_pytest.log 2>&1; echo "pytest rc $?" >> $O/ar_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/ar_smoke.log 2>&1; echo "smoke rc $?" >> $O/ar_smoke.log
export CD_TUNE_CACHE=$O/ar_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/ar_bench.json 2> $O/ar_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/ar_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/ar_bench_ncu.log 2>&1
timeout 600 python bench.py --impl reference > $O/ar_bench_ref.json 2> $O/ar_bench_ref.err
tail -3 $O/ar_pytest.log; tail -3 $O/ar_smoke.log
python -c "import json; d=json.load(open('$O/ar_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['e2e'], d['clocks'], d['roofline'], d['also'].get('2^4_fp32_chain'))"
head -c 400 $O/ar_bench_ref.json
