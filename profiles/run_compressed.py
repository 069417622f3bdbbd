"""Full (9-matrix) vs hermiticity-compressed (5-matrix) links (fp32 or --prec fp16), tau3-hermitian operator.
python profiles/run_compressed.py --dims 8 8 8 8 --nvec 24"""
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
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--json", default=None)
ap.add_argument("--prec", default="fp32")
ap.add_argument("--mask", type=int, default=0, help="CD_OPT_HALO_SELF_MASK (multi-rank path on one GPU)")
a = ap.parse_args()
dims = tuple(a.dims)
V = dims[0] * dims[1] * dims[2] * dims[3]
N = 2 * a.nvec
ctx = cd.Context(dims, a.nvec)
if a.mask:
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, a.mask)
L = ctx.links_generate(a.prec, kind="hermitian", scale_log2=-4)
C, dev = L.compress_hermitian()
x, y = ctx.field(a.prec), ctx.field(a.prec)
x.generate()
s = torch.cuda.current_stream()


def timed(links):
    for _ in range(5):
        links.apply(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    u, w = x, y
    for _ in range(a.reps):
        links.apply(w, u)
        u, w = w, u
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps * 1e3


t_full, t_comp = timed(L), timed(C)
mb9 = perfmodel.metric_bytes_per_site(a.nvec, a.prec) * V
mrec, vrec = (8 * N * N, 8 * N) if a.prec == "fp32" else (4 * N * N + 16, 4 * N + 16)
mb5 = (5 * mrec + 9 * vrec) * V
row = {"dims": dims, "nvec": a.nvec, "prec": a.prec, "halo_mask": a.mask, "max_dev": dev, "us_full": round(t_full, 2), "us_compressed": round(t_comp, 2),
       "speedup": round(t_full / t_comp, 3), "full_GBs": round(mb9 / t_full / 1e3, 1),
       "compressed_GBs_5matrix_bytes": round(mb5 / t_comp / 1e3, 1),
       "compressed_GBs_9matrix_equiv": round(mb9 / t_comp / 1e3, 1),
       "variant_full": ctx.variants(a.prec)[ctx.chosen_variant(a.prec)]}
print(json.dumps(row), flush=True)
if a.json:
    open(a.json, "a").write(json.dumps(row) + "\n")
