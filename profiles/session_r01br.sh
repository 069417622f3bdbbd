#!/bin/bash
# Round-1 session br: bench with the tuner's near-tie rule (8^4 fp32 should pick a TMA ring); parity of the apply path.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "all_variants or graph or full_size" > $O/br_pytest.log 2>&1; echo "pytest rc $?" >> $O/br_pytest.log
export CD_TUNE_CACHE=$O/br_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/br_bench.json 2> $O/br_bench.err
tail -2 $O/br_pytest.log; cat $CD_TUNE_CACHE
python -c "import json; d=json.load(open('$O/br_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], d['also']['2^4_fp32_chain']['us_per_apply'], d['also']['2^4_fp32_chain']['pct_of_8tbs'])"
