#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
for cfg in "orig 3" "split3 3" "split3 2"; do
 set -- $cfg
 CD_MRHS_NBS=$2 CD_LIB_PATH=ab_libs/mrhs_$1.so timeout 300 python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 128 --reps 20 2>&1 | tail -1 | cut -c1-120 | sed "s/^/$1 nbs=$2 8^4 nv24: /" >> gpurun_out/r02w2_mrhs.txt
 CD_MRHS_NBS=$2 CD_LIB_PATH=ab_libs/mrhs_$1.so timeout 300 python profiles/run_mrhs.py --dims 6 6 6 12 --nvec 32 --nrhs 128 --reps 20 2>&1 | tail -1 | cut -c1-120 | sed "s/^/$1 nbs=$2 M4 nv32: /" >> gpurun_out/r02w2_mrhs.txt
done
done
CD_LIB_PATH=ab_libs/mrhs_split3.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mrhs" > gpurun_out/r02w2_parity.log 2>&1
echo "parity rc=$?"
cat gpurun_out/r02w2_mrhs.txt
