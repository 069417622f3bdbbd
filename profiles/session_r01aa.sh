#!/bin/bash
# Round-1 session aa: bench with the grouped e2e pipeline (tune cache written), then the ncu launch
# list of the same command reading that tune cache (so the launched kernels match the timed run).
O=gpurun_out
export CD_TUNE_CACHE=$O/aa_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/aa_bench.json 2> $O/aa_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/aa_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/aa_bench_ncu.log 2>&1
cat $CD_TUNE_CACHE
python -c "import json; d=json.load(open('$O/aa_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['e2e'], d['clocks'], d['also']['2^4_fp32_chain'])"
