#!/bin/bash
# Round-1 session y: A/B of the link-load cache hint (.L2::256B prefetch) on the single-apply kernels.
O=gpurun_out
: > $O/y_ab.txt
for rep in 1 2; do
for lib in libcoarse_dslash libcd_hint1; do
  echo "== $lib rep $rep" >> $O/y_ab.txt
  CD_LIB_PATH=paper_1612_07873_b200/$lib.so timeout 300 python profiles/run_apply.py --sweep --dims 8 8 8 8 --nvec 24 --prec fp32 >> $O/y_ab.txt 2>&1
  CD_LIB_PATH=paper_1612_07873_b200/$lib.so timeout 300 python profiles/run_apply.py --sweep --dims 8 8 8 8 --nvec 24 --prec fp16 >> $O/y_ab.txt 2>&1
  CD_LIB_PATH=paper_1612_07873_b200/$lib.so timeout 300 python profiles/run_apply.py --sweep --dims 16 16 16 8 --nvec 24 --prec fp16 >> $O/y_ab.txt 2>&1
done; done
cat $O/y_ab.txt | grep -v "^$" | awk '{print $1, $2, $3, $5, $6}' | head -150
