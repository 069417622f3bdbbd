#!/bin/bash
# Round-1 session bw: final bench line (tune cache written), launch list of the same command, reference arm.
O=gpurun_out
export CD_TUNE_CACHE=$O/bw_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/bw_bench.json 2> $O/bw_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/bw_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/bw_bench_ncu.log 2>&1
timeout 600 python bench.py --impl reference > $O/bw_bench_ref.json 2> $O/bw_bench_ref.err
cat $CD_TUNE_CACHE
python -c "import json; d=json.load(open('$O/bw_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['e2e']['value'], d['clocks'], d['roofline'], d['also']['2^4_fp32_chain'], d['cpu_baseline']['value'])"
