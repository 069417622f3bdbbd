#!/bin/bash
# Round-1 session as: the tuner times variants back-to-back with the production PDL setting -- bench.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "all_variants or graph or tuner or full_size" > $O/as_pytest.log 2>&1; echo "pytest rc $?" >> $O/as_pytest.log
export CD_TUNE_CACHE=$O/as_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/as_bench.json 2> $O/as_bench.err
timeout 600 python bench.py --prec fp16 --no-cpu --no-extras > $O/as_bench16.json 2> $O/as_bench16.err
tail -2 $O/as_pytest.log; cat $CD_TUNE_CACHE
python -c "import json; d=json.load(open('$O/as_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['clocks'], d['roofline']['frac'])"
python -c "import json; d=json.load(open('$O/as_bench16.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['clocks'], d['roofline']['frac'])"
