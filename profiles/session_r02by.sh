#!/bin/bash
# round 2, session by: A/B of two builds on one box -- HEAD (consumers quantise, store_site) vs the dedicated
# fp16 epilogue warp -- swapping the in-tree .so between interleaved rounds (profiles/ab/lib_{head,new}.so)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
O=gpurun_out/r02by_epw_ab.txt
LIB=paper_1612_07873_b200/libcoarse_dslash.so
for r in 1 2 3; do
 for v in head new; do
  cp profiles/ab/lib_$v.so $LIB
  echo "== $v round $r" >> $O
  timeout 300 python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 10 --secs 0.6 --rounds 2 >> $O 2>&1
  timeout 300 python profiles/ring_sustained.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variants 10 --secs 0.4 --rounds 2 >> $O 2>&1
  timeout 300 python profiles/ring_sustained.py --dims 6 6 6 12 --nvec 32 --prec fp16 --variants 8 --secs 0.4 --rounds 2 >> $O 2>&1
 done
done
cp profiles/ab/lib_new.so $LIB
cat $O
