#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
for lib in nodirect direct; do
 for d in "2 2 2 2" "4 4 4 4"; do
  for p in fp32 fp16; do
   CD_LIB_PATH=ab_libs/$lib.so timeout 300 python profiles/run_apply.py --dims $d --nvec 24 --prec $p --sweep --graph 2>&1 | grep fg_kw1 | sed "s/^/$lib /" >> gpurun_out/r02ah_direct.txt
  done
 done
done
done
CD_LIB_PATH=ab_libs/direct.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "all_variants or random or impulse or shift" > gpurun_out/r02ah_parity.log 2>&1
echo "parity rc=$?"
tail -2 gpurun_out/r02ah_parity.log
