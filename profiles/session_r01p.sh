#!/bin/bash
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "mrhs" 2>&1 | grep -E "^E |passed|failed" | head -5
for d in "4 4 4 4" "8 8 8 8"; do
  python profiles/run_mrhs.py --dims $d --nvec 24 --nrhs 128 --json $O/mrhs_p.jsonl
done
python profiles/run_mrhs.py --dims 6 6 6 12 --nvec 32 --nrhs 128 --json $O/mrhs_p.jsonl
