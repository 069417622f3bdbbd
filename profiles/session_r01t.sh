#!/bin/bash
# Round-1 session t: ncu DRAM validation of BASELINE configs M4 (6^3x12, Nvec 32, fp32) and
# M5 (16^3x32, Nvec 24, fp16) with the autotuned variant, cold (--cache-control all), one launch.
O=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
ncu --metrics $M --clock-control none -k regex:dslash -s 300 -c 1 --csv --log-file $O/ncu_m4.csv \
    python profiles/run_apply.py --dims 6 6 6 12 --nvec 32 --prec fp32 --reps 400 > $O/m4.log 2>&1
ncu --metrics $M --clock-control none -k regex:dslash -s 300 -c 1 --csv --log-file $O/ncu_m5.csv \
    python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --reps 400 > $O/m5.log 2>&1
python profiles/run_apply.py --dims 6 6 6 12 --nvec 32 --prec fp32 --reps 200 >> $O/m4.log 2>&1
python profiles/run_apply.py --dims 16 16 16 32 --nvec 24 --prec fp16 --reps 20 >> $O/m5.log 2>&1
tail -n 3 $O/m4.log $O/m5.log
