#!/bin/bash
# Round-1 session ay: ncu --set full + source page of the 2000-apply launch of the cluster push chain (variant 4000, 2^4).
O=gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dslash_cpush --launch-skip 1 -c 1 -o $O/ay_cpush \
  python profiles/run_chain_prof.py --variant 4000 --n 2000 > $O/ay_ncu.log 2>&1
ncu -i $O/ay_cpush.ncu-rep --page source --csv --print-source sass > $O/ay_cpush_source.csv 2>/dev/null
ncu -i $O/ay_cpush.ncu-rep --page raw --csv > $O/ay_cpush_raw.csv 2>/dev/null
tail -3 $O/ay_ncu.log
