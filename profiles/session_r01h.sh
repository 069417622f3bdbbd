#!/bin/bash
# Round-1 session h: bench lines (ours fp32/fp16, reference arm), ncu launch list of the bench,
# ncu --set full of the tuned 8^4 kernels, hot-state DRAM bytes (cache-control none).
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/gpu.txt
python bench.py > $O/bench_fp32.json 2> $O/bench_fp32.err
python bench.py --prec fp16 --no-cpu > $O/bench_fp16.json 2> $O/bench_fp16.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file $O/launches_bench_r01.csv python bench.py --steps 20 --warmup 3 --no-cpu > $O/bench_under_ncu.log 2>&1
V32=$(python -c "import json;print(json.load(open('$O/bench_fp32.json'))['config']['variant'])")
V16=$(python -c "import json;print(json.load(open('$O/bench_fp16.json'))['config']['variant'])")
echo "tuned: $V32 $V16" > $O/tuned.txt
python - <<PY > $O/ids.txt
import paper_1612_07873_b200 as cd
c = cd.Context((8,8,8,8), 24)
print(c.variants('fp32').index('$V32'), c.variants('fp16').index('$V16'))
PY
read I32 I16 < $O/ids.txt
ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/prof_r01_8444_f32 \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant $I32 --reps 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dslash -s 4 -c 1 -f -o $O/prof_r01_8444_f16 \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp16 --variant $I16 --reps 6 > /dev/null 2>&1
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:dslash -s 20 -c 10 --csv --log-file $O/hot_dram_f32.csv \
    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant $I32 --reps 40 > /dev/null 2>&1
ls -la $O
