#!/bin/bash
# Round-1 session aq: ring prefetches the link copies of as many static sites as the ring holds before
# griddepcontrol.wait -- parity of every variant, then A/B/C timing (original / one site / ring-full).
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "all_variants or halo_self or full_size or impulse or shift or identity or graph" > $O/aq_pytest.log 2>&1; echo "pytest rc $?" >> $O/aq_pytest.log
for rep in 1 2; do
for lib in build_ab/lib_before_ringpre.so build_ab/lib_ringpre1.so paper_1612_07873_b200/libcoarse_dslash.so; do
  tag=$(basename $lib .so)
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 8 8 8 8 --prec fp16 --reps 40 --tag $tag >> $O/aq_ab.jsonl 2>> $O/aq_ab.err
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 8 8 8 8 --prec fp32 --reps 40 --tag $tag >> $O/aq_ab.jsonl 2>> $O/aq_ab.err
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 16 16 16 32 --prec fp16 --reps 4 --tag $tag >> $O/aq_ab.jsonl 2>> $O/aq_ab.err
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/ring_ab.py --dims 6 6 6 12 --nvec 32 --prec fp32 --reps 40 --tag $tag >> $O/aq_ab.jsonl 2>> $O/aq_ab.err
done
done
tail -2 $O/aq_pytest.log; python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/aq_ab.jsonl"):
    r = json.loads(l); d[(tuple(r["dims"]), r["prec"], r["variant"], r["tag"])].append(r["us"])
for k in sorted(d): print(k, min(d[k]))
PY
