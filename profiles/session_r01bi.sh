#!/bin/bash
# Round-1 session bi: cluster push chain -- one barrier per producer triple (a thread waits only for the
# producer triple that owns its chunk) vs one per kind; parity, sanitizers, A/B.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain_tuner" > $O/bi_pytest.log 2>&1; echo "pytest rc $?" >> $O/bi_pytest.log
for tool in racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 4000 > $O/bi_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bi_san_$tool.log
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 3 1 5 1 4000 >> $O/bi_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bi_san_$tool.log
done
for rep in 1 2 3; do
for lib in build_ab/lib_cpush_head.so build_ab/lib_cpush_pertriple.so; do
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 2>> $O/bi.err | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" >> $O/bi.jsonl
done
done
tail -2 $O/bi_pytest.log; grep -h "rc \|SUMMARY" $O/bi_san_*.log
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/bi.jsonl"):
    r = json.loads(l); d[(r["lib"], r["variant"])].append(r["us_med"])
for k in sorted(d): print(k, d[k])
PY
