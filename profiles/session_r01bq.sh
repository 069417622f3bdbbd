#!/bin/bash
# Round-1 session bq: 8^4 fp32 bench under sustained (power-capped) load -- fg_kw3_wr4 vs ring_tma_m1/m3, twice.
O=gpurun_out
python - <<'PY' > $O/bq_ids.txt
import paper_1612_07873_b200 as cd
ctx = cd.Context((8, 8, 8, 8), 24)
for i, n in enumerate(ctx.variants("fp32")): print(i, n)
PY
cat $O/bq_ids.txt
R1=$(grep ring_tma_m1_f32 $O/bq_ids.txt | cut -d' ' -f1); R3=$(grep ring_tma_m3_f32 $O/bq_ids.txt | cut -d' ' -f1); FG=$(grep fg_kw3_wr4_f32 $O/bq_ids.txt | cut -d' ' -f1)
for rep in 1 2; do
for v in $FG $R1 $R3; do
  CD_VARIANT=$v timeout 600 python bench.py --no-cpu --no-extras > $O/bq_${v}_${rep}.json 2>> $O/bq.err
  python -c "import json; d=json.load(open('$O/bq_${v}_${rep}.json')); print('variant $v', d['config']['variant'], d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
