import os, sys
sys.path.insert(0, "/root/repo")
os.environ.setdefault("CD_TUNE", "0")
import torch
import paper_1612_07873_b200 as cd
for prec in ("fp32", "fp16"):
    ctx = cd.Context((8, 8, 4, 5), 24)
    L = ctx.links_generate(prec, scale_log2=-4)
    a, b = ctx.field(prec), ctx.field(prec)
    a.generate()
    for v, n in enumerate(ctx.variants(prec)):
        if n.startswith("ring"):
            ctx.set_option(cd.CD_OPT_VARIANT, v)
            L.apply(b, a)
torch.cuda.synchronize()
print("ring race run ok")
