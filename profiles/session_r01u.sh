#!/bin/bash
# Round-1 session u (after container restore): full GPU test suite, smoke, default bench line,
# reference arm, launch list of the bench command.
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/u_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/u_pytest.log 2>&1; echo "pytest rc=$?" >> $O/u_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/u_smoke.log 2>&1; echo "smoke rc=$?" >> $O/u_smoke.log
timeout 600 python bench.py > $O/u_bench.json 2> $O/u_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/u_bench_ref.json 2> $O/u_bench_ref.err
tail -n 3 $O/u_pytest.log $O/u_smoke.log; cat $O/u_bench.json
