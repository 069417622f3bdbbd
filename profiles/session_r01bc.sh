#!/bin/bash
# Round-1 session bc: cluster push chain -- early remote arrive.expect_tx (off the epilogue); parity, sanitizers, A/B.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cpush or chain_tuner" > $O/bc_pytest.log 2>&1; echo "pytest rc $?" >> $O/bc_pytest.log
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 2 2 2 2 4000 > $O/bc_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bc_san_$tool.log
timeout 600 compute-sanitizer --tool $tool --error-exitcode=3 python profiles/cpush_debug.py 3 1 5 1 4000 >> $O/bc_san_$tool.log 2>&1; echo "$tool rc $?" >> $O/bc_san_$tool.log
done
for rep in 1 2 3; do
for lib in build_ab/lib_cpush_triple.so build_ab/lib_cpush_early.so; do
  CD_LIB_PATH=$PWD/$lib timeout 300 python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 --variants 4000 3002 2>> $O/bc.err | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" >> $O/bc.jsonl
done
done
tail -2 $O/bc_pytest.log; grep -h "rc \|SUMMARY" $O/bc_san_*.log
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/bc.jsonl"):
    r = json.loads(l); d[(r["lib"], r["variant"])].append(r["us_med"])
for k in sorted(d): print(k, d[k])
PY
