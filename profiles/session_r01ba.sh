#!/bin/bash
# Round-1 session ba: cluster push chain A/B -- per-triple named barrier vs one CTA barrier (2^4, Nvec 24).
O=gpurun_out
for rep in 1 2 3; do
for lib in build_ab/lib_cpush_triple.so build_ab/lib_cpush_ctabar.so; do
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 2>> $O/ba.err | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" >> $O/ba.jsonl
done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ba.jsonl"):
    r = json.loads(l); d[(r["lib"], r["variant"])].append(r["us_med"])
for k in sorted(d): print(k, d[k])
PY
