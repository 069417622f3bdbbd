#!/bin/bash
O=gpurun_out
python profiles/run_compressed.py --dims 8 8 8 8 --nvec 24 --json $O/comp.jsonl
python profiles/run_compressed.py --dims 6 6 6 12 --nvec 32 --json $O/comp.jsonl
python profiles/run_compressed.py --dims 16 16 16 8 --nvec 24 --reps 40 --json $O/comp.jsonl
python profiles/run_compressed.py --dims 4 4 4 4 --nvec 24 --json $O/comp.jsonl
ncu --set full --clock-control none --import-source on -k regex:fgh -s 4 -c 1 -f -o $O/prof_fgh \
    python profiles/run_compressed.py --dims 8 8 8 8 --nvec 24 --reps 5 > /dev/null 2>&1
ls $O/prof_fgh.ncu-rep
