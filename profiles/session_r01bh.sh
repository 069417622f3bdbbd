#!/bin/bash
# Round-1 session bh: ncu --set full + source page of the 2000-apply launch of the final cluster push chain (variant 4000, 2^4).
O=gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dslash_cpush --launch-skip 1 -c 1 -o $O/bh_cpush \
  python profiles/run_chain_prof.py --variant 4000 --n 2000 > $O/bh_ncu.log 2>&1
ncu -i $O/bh_cpush.ncu-rep --page source --csv --print-source sass > $O/bh_cpush_source.csv 2>/dev/null
ncu -i $O/bh_cpush.ncu-rep --page raw --csv > $O/bh_cpush_raw.csv 2>/dev/null
tail -3 $O/bh_ncu.log
