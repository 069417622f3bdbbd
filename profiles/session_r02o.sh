#!/bin/bash
# round 2, session o: split vs unsplit under sustained load (PDL effect), M1/M2 graph PDL on/off
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python profiles/split_sustained.py --mask 8 --secs 1.0 --rounds 3 > gpurun_out/r02o_split_sustained.txt 2>&1
timeout 600 python profiles/split_sustained.py --mask 12 --secs 1.0 --rounds 2 >> gpurun_out/r02o_split_sustained.txt 2>&1
for pdl in 1 0; do
 for d in "2 2 2 2" "4 4 4 4"; do
  CD_PDL=$pdl timeout 300 python profiles/run_apply.py --dims $d --nvec 24 --prec fp32 --sweep --graph 2>&1 | sed "s/^/pdl=$pdl /" >> gpurun_out/r02o_graph_pdl.txt
 done
done
cat gpurun_out/r02o_split_sustained.txt
