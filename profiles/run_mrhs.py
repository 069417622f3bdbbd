"""Time the tcgen05 multi-RHS apply (coarse_dslash_apply_mrhs) and the single-RHS fp16 apply
for comparison.  python profiles/run_mrhs.py --dims 8 8 8 8 --nvec 24 --nrhs 128"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402
import perfmodel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[8, 8, 8, 8])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--nrhs", type=int, default=128)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--json", default=None)
ap.add_argument("--mask", type=int, default=0, help="CD_OPT_HALO_SELF_MASK (multi-rank path on one GPU)")
a = ap.parse_args()
dims = tuple(a.dims)
V = dims[0] * dims[1] * dims[2] * dims[3]
N = 2 * a.nvec
ctx = cd.Context(dims, a.nvec)
if a.mask:
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, a.mask)
L = ctx.links_generate("fp16", scale_log2=-4)
x, y = ctx.field("fp16", nrhs=a.nrhs), ctx.field("fp16", nrhs=a.nrhs)
x.generate()
s = torch.cuda.current_stream()
for _ in range(3):
    L.apply_mrhs(y, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(a.reps):
    L.apply_mrhs(y, x)
e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / a.reps * 1e3
flops = perfmodel.flops_per_site(a.nvec) * V * a.nrhs
link_b = V * 9 * (4 * N * N + 16)
vec_b = V * a.nrhs * (4 * N + 16)
comp = link_b + 2 * vec_b          # links + one read + one write of every vector record
metric = V * perfmodel.metric_bytes_per_site(a.nvec, "fp16") * a.nrhs   # BJ formula per rhs
row = {"dims": dims, "nvec": a.nvec, "nrhs": a.nrhs, "halo_mask": a.mask, "us": round(us, 2), "TFLOPS": round(flops / us / 1e6, 2),
       "compulsory_GBs": round(comp / us / 1e3, 1), "us_per_rhs": round(us / a.nrhs, 4),
       "single_rhs_equiv_GBs": round(metric / us / 1e3, 1)}
print(json.dumps(row), flush=True)
if a.json:
    open(a.json, "a").write(json.dumps(row) + "\n")
