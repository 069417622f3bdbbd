"""Time every apply_chain variant on a small lattice (µs per apply, CUDA events around one
launch of n chained applies) and sanity-check each against single applies.
python profiles/run_chain_sweep.py --dims 2 2 2 2 --nvec 24 --n 2000 [--trace out.bin]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[2, 2, 2, 2])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp32")
ap.add_argument("--n", type=int, default=800)   # links x 2^-4 grow the iterate ~1.09x per apply: 800 stays finite
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--variants", type=int, nargs="*", default=None)
ap.add_argument("--trace", default=None, help="dump the CTA-0 trace of --trace-variant here")
ap.add_argument("--trace-variant", type=int, default=3001)
ap.add_argument("--poll-ns", type=int, default=0, help="CD_POLL_NS for the chain kernels")
ap.add_argument("--d0", type=int, default=None, help="CD_POLL_D0 (cycles) for the LL-register chain")
ap.add_argument("--d1", type=int, default=None, help="CD_POLL_D1 (cycles) for the LL-register chain")
a = ap.parse_args()
if a.poll_ns:
    os.environ["CD_POLL_NS"] = str(a.poll_ns)
if a.d0 is not None:
    os.environ["CD_POLL_D0"] = str(a.d0)
if a.d1 is not None:
    os.environ["CD_POLL_D1"] = str(a.d1)
ctx = cd.Context(tuple(a.dims), a.nvec)
L = ctx.links_generate(a.prec, scale_log2=-4)
x, y = ctx.field(a.prec), ctx.field(a.prec)
x.generate()
v0 = x.export()
# reference: 5 single applies with the tuned single-apply kernel
r0, r1 = ctx.field(a.prec), ctx.field(a.prec)
r0.import_(v0)
for _ in range(5):
    L.apply(r1, r0)
    r0, r1 = r1, r0
ref = r0.export()
names = ctx.variants(a.prec)
cands = a.variants if a.variants else [5000, 4000, 1000, 1001] + [2000 + i for i in range(1, len(names))] + list(range(3001, 3007))
V = int(np.prod(a.dims))
rows = []
for vid in cands:
    ctx.set_option(cd.CD_OPT_VARIANT, vid)
    x.import_(v0)
    try:
        L.apply_chain(x, y, 5)
    except cd.CDError as e:
        continue
    got = y.export()
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    L.apply_chain(x, y, 8)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        x.import_(v0)   # untimed: every timed launch starts from the same finite vector
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)   # keeps the stream busy while the host submits (no idle in the window)
        e0.record()
        L.apply_chain(x, y, a.n)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / a.n)
    name = names[vid - 2000] if 2000 <= vid < 3000 else (names[vid] if vid < 1000 else
                                                         {1000: "cluster", 1001: "push"}.get(vid, str(vid)))
    r = {"dims": a.dims, "nvec": a.nvec, "prec": a.prec, "variant": vid, "name": name,
         "poll_ns": a.poll_ns, "d0": a.d0, "d1": a.d1, "us_min": round(min(ts), 4), "us_med": round(float(np.median(ts)), 4), "rel_vs_single": err}
    rows.append(r)
    print(json.dumps(r), flush=True)
if a.trace:
    ctx.set_option(cd.CD_OPT_VARIANT, a.trace_variant)
    os.environ["CD_CHAIN_TRACE"] = a.trace
    x.import_(v0)
    L.apply_chain(x, y, 1024)
    torch.cuda.synchronize()
    del os.environ["CD_CHAIN_TRACE"]
ctx.set_option(cd.CD_OPT_VARIANT, -1)
