#!/bin/bash
# round 2, session br: compressed ring (NEXT-2) with one copy for the site's own five records and gather4 vectors
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compress" > gpurun_out/r02br_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r02br_parity.log
O=gpurun_out/r02br_comp.txt
for g in 1 0 1; do
 for m in 3 9; do
  echo "== CD_RING_GATHER=$g CD_COMP_MPS=$m" >> $O
  CD_RING_GATHER=$g CD_COMP_MPS=$m timeout 300 python profiles/run_compressed_ab.py --dims 16 16 16 32 --prec fp16 --secs 0.6 >> $O 2>&1
 done
 echo "== CD_RING_GATHER=$g 8^4 fp16" >> $O
 CD_RING_GATHER=$g timeout 300 python profiles/run_compressed_ab.py --dims 8 8 8 8 --prec fp16 --secs 0.4 >> $O 2>&1
 echo "== CD_RING_GATHER=$g 8^4 fp32 ring" >> $O
 CD_COMP_RING=1 CD_RING_GATHER=$g timeout 300 python profiles/run_compressed_ab.py --dims 8 8 8 8 --prec fp32 --secs 0.4 >> $O 2>&1
done
cat $O
