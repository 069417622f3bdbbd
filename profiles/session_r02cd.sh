#!/bin/bash
# round 2, session cd: parity after removing the two-group ring machinery; quick bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r02cd_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/r02cd_parity.log
timeout 600 python bench.py --no-extras > gpurun_out/r02cd_bench.json 2> gpurun_out/r02cd_bench.err
echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02cd_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
