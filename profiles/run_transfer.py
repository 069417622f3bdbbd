"""Restrictor / prolongator bandwidth.  Algorithmic bytes per launch:
restrict = basis (8 nf Nvec per fine site) + fine vector read (8 nf) + coarse write (8 N per coarse site);
prolong  = basis + fine vector write + coarse read.
python profiles/run_transfer.py --cdims 8 8 8 8 --block 4 4 4 4 --nspin 4 --ncolor 3 --nvec 24"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cdims", type=int, nargs=4, default=[8, 8, 8, 8])
ap.add_argument("--block", type=int, nargs=4, default=[4, 4, 4, 4])
ap.add_argument("--nspin", type=int, default=4)
ap.add_argument("--ncolor", type=int, default=3)
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp32")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--json", default=None)
a = ap.parse_args()
ctx = cd.Context(tuple(a.cdims), a.nvec)
nf = a.nspin * a.ncolor
Vc = ctx.V
Vf = Vc * int(torch.tensor(a.block).prod())
W = torch.randn(Vf, a.nspin, a.ncolor, a.nvec, dtype=torch.complex64, device="cuda")
T = ctx.transfer(a.block, a.nspin, a.ncolor, W)
del W
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.current_stream()
e0.record(s)
T.orthonormalise()
e1.record(s)
torch.cuda.synchronize()
ortho_ms = e0.elapsed_time(e1)
fine = torch.randn(Vf, a.nspin, a.ncolor, dtype=torch.complex64, device="cuda")
fine2 = torch.empty_like(fine)
c = ctx.field(a.prec)


def timed(fn):
    """reps launches captured in one CUDA graph (no Python launch overhead in the timing)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(a.reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps * 1e3


t_r = timed(lambda: T.restrict(c, fine))
t_p = timed(lambda: T.prolong(fine2, c))
wb = Vf * nf * a.nvec * 8
vb = Vf * nf * 8
cb = Vc * 2 * a.nvec * (8 if a.prec == "fp32" else 4) + (0 if a.prec == "fp32" else 16 * Vc)
row = {"cdims": a.cdims, "block": a.block, "nspin": a.nspin, "ncolor": a.ncolor, "nvec": a.nvec, "prec": a.prec,
       "basis_MB": round(wb / 1e6, 1), "orthonormalise_ms": round(ortho_ms, 2),
       "us_restrict": round(t_r, 2), "us_prolong": round(t_p, 2),
       "restrict_GBs": round((wb + vb + cb) / t_r / 1e3, 1), "prolong_GBs": round((wb + vb + cb) / t_p / 1e3, 1)}
print(json.dumps(row), flush=True)
if a.json:
    open(a.json, "a").write(json.dumps(row) + "\n")
