#!/bin/bash
O=gpurun_out
for ns in 0 20 50 100 200; do
  echo "poll_ns=$ns"
  CD_POLL_NS=$ns python profiles/run_apply.py --sweep --dims 2 2 2 2 --nvec 24 --prec fp32 --chain 2>&1 | grep -E "ll_fg_kw1_wr1|ll_fg_kw3_wr2|ll_fg_kw9_wr3"
  CD_POLL_NS=$ns python profiles/run_apply.py --sweep --dims 2 2 2 2 --nvec 24 --prec fp16 --chain 2>&1 | grep -E "ll_fg"
done
