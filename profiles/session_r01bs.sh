#!/bin/bash
# Round-1 session bs: ncu --set full of ring_tma_m3 / ring_tma_m1 fp32 at 8^4 (the tuner's pick after the
# near-tie rule; both carry the first-site prefetch now) -> traffic for bench.py; launch list of the bench command.
O=gpurun_out
for v in 10 0; do
  ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/bs_f32_v$v \
      python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant $v --reps 6 > /dev/null 2>&1
  ncu -i $O/bs_f32_v$v.ncu-rep --page raw --csv > $O/bs_f32_v$v.raw.csv 2>/dev/null
done
export CD_TUNE_CACHE=$O/bs_tune.txt
rm -f $CD_TUNE_CACHE
timeout 600 python bench.py > $O/bs_bench.json 2> $O/bs_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/bs_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/bs_bench_ncu.log 2>&1
cat $CD_TUNE_CACHE
python - <<'PY'
import csv
for v in (10, 0):
    rows = list(csv.reader(open(f"gpurun_out/bs_f32_v{v}.raw.csv")))
    h, vals = rows[0], rows[2]
    d = dict(zip(h, vals))
    print(v, d.get("Kernel Name", "")[:40], d["gpu__time_duration.sum"], d["dram__bytes_read.sum"], d["dram__bytes_write.sum"])
PY
python -c "import json; d=json.load(open('gpurun_out/bs_bench.json')); print(d['value'], d['ms_per_step'], d['config']['variant'], d['clocks'], d['roofline'])"
