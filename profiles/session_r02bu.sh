#!/bin/bash
# round 2, session bu: gather4 for face sites' local blocks on split contexts: parity + fused split A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "halo or multirank or gather4 or split or fullsize or whole" > gpurun_out/r02bu_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r02bu_parity.log
O=gpurun_out/r02bu_split_gather.txt
for d in "16 16 16 4" "16 16 16 16" "16 16 16 32"; do
  set -- $d
  timeout 300 python profiles/split_gather_ab.py --dims $1 $2 $3 $4 >> $O 2>&1
done
cat $O
