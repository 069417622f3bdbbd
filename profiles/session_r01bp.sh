#!/bin/bash
# Round-1 session bp: final GPU check (suite, smoke, bench with the 800-apply chain protocol, launch list, reference arm).
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/bp_pytest.log 2>&1; echo "pytest rc $?" >> $O/bp_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/bp_smoke.log 2>&1; echo "smoke rc $?" >> $O/bp_smoke.log
export CD_TUNE_CACHE=$O/bp_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/bp_bench.json 2> $O/bp_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/bp_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/bp_bench_ncu.log 2>&1
timeout 600 python bench.py --impl reference > $O/bp_bench_ref.json 2> $O/bp_bench_ref.err
tail -3 $O/bp_pytest.log; tail -3 $O/bp_smoke.log
python -c "import json; d=json.load(open('$O/bp_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['e2e'], d['clocks'], d['roofline'], d['also'].get('2^4_fp32_chain'))"
head -c 400 $O/bp_bench_ref.json
