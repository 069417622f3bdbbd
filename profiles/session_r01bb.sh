#!/bin/bash
# Round-1 session bb: cluster push chain -- two-level reduce-scatter (the lane-pair sum moves into the triple's
# shared-memory reduction) vs three-level; parity + A/B.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush" > $O/bb_pytest.log 2>&1; echo "pytest rc $?" >> $O/bb_pytest.log
for rep in 1 2 3; do
for lib in build_ab/lib_cpush_triple.so build_ab/lib_cpush_rs2.so; do
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 2>> $O/bb.err | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" >> $O/bb.jsonl
done
done
tail -2 $O/bb_pytest.log
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/bb.jsonl"):
    r = json.loads(l); d[(r["lib"], r["variant"])].append(r["us_med"])
for k in sorted(d): print(k, d[k])
PY
