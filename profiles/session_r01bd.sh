#!/bin/bash
# Round-1 session bd: cluster push chain A/B/C -- early arrive (committed) / + output sign folded into the
# links / + 16-B row-pair pushes; parity of the candidates through CD_LIB_PATH.
O=gpurun_out
for lib in build_ab/lib_cpush_fold.so build_ab/lib_cpush_p16.so; do
  CD_LIB_PATH=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush" > $O/bd_pytest_$(basename $lib .so).log 2>&1; echo "pytest rc $?" >> $O/bd_pytest_$(basename $lib .so).log
done
for rep in 1 2 3; do
for lib in build_ab/lib_cpush_early.so build_ab/lib_cpush_fold.so build_ab/lib_cpush_p16.so; do
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 2>> $O/bd.err | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" >> $O/bd.jsonl
done
done
tail -1 $O/bd_pytest_*.log
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/bd.jsonl"):
    r = json.loads(l); d[(r["lib"], r["variant"])].append(r["us_med"])
for k in sorted(d): print(k, d[k])
PY
