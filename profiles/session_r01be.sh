#!/bin/bash
# Round-1 session be: full GPU suite + smoke + bench (tune cache written) + ncu launch list of the same bench command.
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/be_pytest.log 2>&1; echo "pytest rc $?" >> $O/be_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/be_smoke.log 2>&1; echo "smoke rc $?" >> $O/be_smoke.log
export CD_TUNE_CACHE=$O/be_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/be_bench.json 2> $O/be_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/be_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/be_bench_ncu.log 2>&1
timeout 600 python bench.py --impl reference > $O/be_bench_ref.json 2> $O/be_bench_ref.err
tail -3 $O/be_pytest.log; tail -3 $O/be_smoke.log
python -c "import json; d=json.load(open('$O/be_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['e2e'], d['clocks'], d['roofline'], d['also'].get('2^4_fp32_chain'))"
head -c 400 $O/be_bench_ref.json
