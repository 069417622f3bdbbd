#!/bin/bash
# Round-1 session s: ncu full captures of the SURVEY §8(f) NEXT-row kernels (one launch each).
O=gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:dslash_parity -s 4 -c 2 -o $O/prof_eo_8444 python profiles/run_eo.py --dims 8 8 8 8 --reps 3 > /dev/null 2>&1
$N -k regex:"restrict_kernel|prolong_kernel" -s 6 -c 2 -o $O/prof_transfer_32to8 python profiles/run_transfer.py --reps 2 > /dev/null 2>&1
$N -k regex:dslash_mrhs -s 2 -c 1 -o $O/prof_mrhs_v2_8444 python profiles/run_mrhs.py --reps 2 > /dev/null 2>&1
$N -k regex:dslash_fgh -s 3 -c 1 -o $O/prof_compressed_8444 python profiles/run_compressed.py --reps 3 > /dev/null 2>&1
ls -la $O
