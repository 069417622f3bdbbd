#!/bin/bash
# Round-1 session bt: ring fp32 consumers on FFMA2 (packed FP32) vs FFMA -- parity, sustained bench A/B (ring_tma_m3 forced).
O=gpurun_out
CD_LIB_PATH=$PWD/build_ab/lib_ring_ffma2.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "all_variants or halo_self or full_size" > $O/bt_pytest.log 2>&1; echo "pytest rc $?" >> $O/bt_pytest.log
for rep in 1 2; do
for lib in build_ab/lib_ring_ffma.so build_ab/lib_ring_ffma2.so; do
  CD_LIB_PATH=$PWD/$lib CD_VARIANT=10 timeout 600 python bench.py --no-cpu --no-extras > $O/bt_$(basename $lib .so)_$rep.json 2>> $O/bt.err
  python -c "import json; d=json.load(open('$O/bt_$(basename $lib .so)_$rep.json')); print('$(basename $lib .so)', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
tail -2 $O/bt_pytest.log
