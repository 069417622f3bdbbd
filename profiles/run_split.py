"""A few applies of one configuration with dims routed through the halo path on one GPU
(CD_OPT_HALO_SELF_MASK), for ncu launch lists: which kernels a split apply launches and how long
each takes alone.   python profiles/run_split.py --dims 16 16 16 32 --nvec 24 --prec fp16 --mask 8 --transport peer"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[16, 16, 16, 32])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp16")
ap.add_argument("--mask", type=int, default=8)
ap.add_argument("--transport", default="peer")
ap.add_argument("--variant", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = cd.Context(tuple(a.dims), a.nvec)
if a.mask:
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, a.mask)
    if a.transport == "peer":
        ctx.peer_connect([ctx.peer_handle()])
    ctx.set_transport(a.transport)
ctx.set_option(cd.CD_OPT_VARIANT, a.variant)
L = ctx.links_generate(a.prec, scale_log2=-4)
x, y = ctx.field(a.prec), ctx.field(a.prec)
x.generate()
for i in range(a.reps):
    L.apply(y, x) if i % 2 == 0 else L.apply(x, y)
torch.cuda.synchronize()
print("variant", ctx.variants(a.prec)[ctx.chosen_variant(a.prec)])
