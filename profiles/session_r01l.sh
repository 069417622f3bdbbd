#!/bin/bash
O=gpurun_out
cat > /tmp/llprof.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_1612_07873_b200 as cd
ctx = cd.Context((2,2,2,2), 24)
L = ctx.links_generate('fp32', scale_log2=-4)
x, y = ctx.field('fp32'), ctx.field('fp32')
x.generate()
ctx.set_option(cd.CD_OPT_VARIANT, 2001)
L.apply_chain(x, y, 4)
L.apply_chain(x, y, 400)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:llchain -s 1 -c 1 -f -o $O/prof_llchain python /tmp/llprof.py > /dev/null 2>&1
ls -la $O/prof_llchain.ncu-rep
