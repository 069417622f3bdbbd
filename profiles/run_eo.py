"""Even-odd Schur operator M_ee (two kernels) vs the full operator, fp32.
python profiles/run_eo.py --dims 8 8 8 8 --nvec 24"""
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
ap.add_argument("--mask", type=int, default=0, help="CD_OPT_HALO_SELF_MASK: route these dims through the halo path")
a = ap.parse_args()
dims = tuple(a.dims)
V = dims[0] * dims[1] * dims[2] * dims[3]
N = 2 * a.nvec
ctx = cd.Context(dims, a.nvec)
if a.mask:
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, a.mask)
L = ctx.links_generate("fp32", kind="general", scale_log2=-4)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
s = torch.cuda.current_stream()
t0.record(s)
E = L.prepare_eo()
t1.record(s)
torch.cuda.synchronize()
prep_ms = t0.elapsed_time(t1)


def timed(fn, x, y):
    for _ in range(5):
        fn(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    u, w = x, y
    for _ in range(a.reps):
        fn(w, u)
        u, w = w, u
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps * 1e3


x, y = ctx.field("fp32"), ctx.field("fp32")
x.generate()
xe, ye = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
xe.import_(torch.randn(V // 2, N, dtype=torch.complex64).numpy())
t_full = timed(L.apply, x, y)
t_eo = timed(E.apply_eo, xe, ye)
mb_full = perfmodel.metric_bytes_per_site(a.nvec, "fp32") * V
# odd kernel: 8 matrices + 8 hop reads + 1 write per odd site; even: 9 + 9 + 1 write + 0 (self is a hop read)
mb_eo = (V // 2) * ((8 + 9) * N * N + (8 + 1 + 9 + 1) * N) * 8
row = {"dims": dims, "nvec": a.nvec, "halo_mask": a.mask, "prepare_ms": round(prep_ms, 2), "us_full": round(t_full, 2),
       "us_schur": round(t_eo, 2), "schur_over_full": round(t_eo / t_full, 3),
       "full_GBs": round(mb_full / t_full / 1e3, 1), "schur_GBs": round(mb_eo / t_eo / 1e3, 1)}
print(json.dumps(row), flush=True)
if a.json:
    open(a.json, "a").write(json.dumps(row) + "\n")
