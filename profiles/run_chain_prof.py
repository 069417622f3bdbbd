"""One coarse_dslash_apply_chain launch (n applies) with a forced chain variant, for ncu.
python profiles/run_chain_prof.py --variant 2001 --n 2000"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[2, 2, 2, 2])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp32")
ap.add_argument("--variant", type=int, default=2001)
ap.add_argument("--n", type=int, default=2000)
a = ap.parse_args()
ctx = cd.Context(tuple(a.dims), a.nvec)
L = ctx.links_generate(a.prec, scale_log2=-4)
x, y = ctx.field(a.prec), ctx.field(a.prec)
x.generate()
ctx.set_option(cd.CD_OPT_VARIANT, a.variant)
L.apply_chain(x, y, 4)
L.apply_chain(x, y, a.n)
torch.cuda.synchronize()
