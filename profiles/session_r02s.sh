#!/bin/bash
# round 2, session s: first-site prefetch in the fused split (pre) vs quad; bench with configs in
# a subprocess; parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for lib in quad pre quad pre; do
  CD_LIB_PATH=ab_libs/$lib.so timeout 600 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 1 | sed "s/^/$lib T /" >> gpurun_out/r02s_split.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_self or fused or all_variants" > gpurun_out/r02s_parity.log 2>&1
echo "parity rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -k "operator and peer" > gpurun_out/r02s_multirank.log 2>&1
echo "multirank rc=$?"
timeout 900 python bench.py > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
echo "bench rc=$?"
cat gpurun_out/r02s_split.txt | cut -c1-120
