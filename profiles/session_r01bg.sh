#!/bin/bash
# Round-1 session bg: cluster push chain A/B -- remote wait ordered after the X math (head) vs not (e1).
O=gpurun_out
for rep in 1 2 3; do
for lib in build_ab/lib_cpush_head.so build_ab/lib_cpush_e1.so; do
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 2>> $O/bg.err | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" >> $O/bg.jsonl
done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/bg.jsonl"):
    r = json.loads(l); d[(r["lib"], r["variant"])].append(r["us_med"])
for k in sorted(d): print(k, d[k])
PY
