#!/bin/bash
# Round-1 session aj: ncu --set full + source page of the cluster push chain (variant 4000, 2^4, 2000 applies).
O=gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dslash_cpush -c 1 -o $O/aj_cpush \
  python profiles/run_chain_prof.py --variant 4000 --n 2000 > $O/aj_ncu.log 2>&1
ncu -i $O/aj_cpush.ncu-rep --page source --csv --print-source sass > $O/aj_cpush_source.csv 2>/dev/null
ncu -i $O/aj_cpush.ncu-rep --page raw --csv > $O/aj_cpush_raw.csv 2>/dev/null
tail -3 $O/aj_ncu.log; ls -la $O/aj_*
