#!/bin/bash
# Round-1 session ab (post-restore): GPU test suite, smoke, bench.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/ab_pytest.log 2>&1; echo "pytest rc $?" >> $O/ab_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/ab_smoke.log 2>&1
timeout 600 python bench.py > $O/ab_bench.json 2> $O/ab_bench.err
tail -3 $O/ab_pytest.log; tail -2 $O/ab_smoke.log; cat $O/ab_bench.json | head -c 600
