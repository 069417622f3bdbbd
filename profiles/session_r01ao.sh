#!/bin/bash
# Round-1 session ao: ring producer issues the first site's link copies before griddepcontrol.wait
# (PDL overlap of the ramp) -- parity of every variant, then A/B timing against the previous library.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "all_variants or halo_self or full_size or impulse or shift or identity or graph" > $O/ao_pytest.log 2>&1; echo "pytest rc $?" >> $O/ao_pytest.log
for rep in 1 2; do
for lib in build_ab/lib_before_ringpre.so paper_1612_07873_b200/libcoarse_dslash.so; do
  tag=$(basename $lib .so)
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 8 8 8 8 --prec fp16 --reps 40 --tag $tag >> $O/ao_ab.jsonl 2>> $O/ao_ab.err
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 8 8 8 8 --prec fp32 --reps 40 --tag $tag >> $O/ao_ab.jsonl 2>> $O/ao_ab.err
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 16 16 16 32 --prec fp16 --reps 4 --tag $tag >> $O/ao_ab.jsonl 2>> $O/ao_ab.err
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 6 6 6 12 --nvec 32 --prec fp32 --reps 40 --tag $tag >> $O/ao_ab.jsonl 2>> $O/ao_ab.err
done
done
tail -3 $O/ao_pytest.log; cat $O/ao_ab.jsonl; tail -3 $O/ao_ab.err
