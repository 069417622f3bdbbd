#!/bin/bash
O=gpurun_out
for d in "2 2 2 2" "4 4 4 4" "8 8 8 8"; do
  python profiles/run_mrhs.py --dims $d --nvec 24 --nrhs 128 --json $O/mrhs.jsonl
done
python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 256 --json $O/mrhs.jsonl
python profiles/run_mrhs.py --dims 6 6 6 12 --nvec 32 --nrhs 128 --json $O/mrhs.jsonl
ncu --set full --clock-control none --import-source on -k regex:mrhs -s 3 -c 1 -f -o $O/prof_mrhs_8444 \
    python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 128 --reps 2 > /dev/null 2>&1
ls $O/prof_mrhs_8444.ncu-rep
