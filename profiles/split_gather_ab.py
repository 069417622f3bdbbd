"""Fused split apply (ring + peer transport, T through the halo path on one GPU) with and without
TMA gather4 for the face sites' local blocks: chained applies in interleaved windows.
    python profiles/split_gather_ab.py --dims 16 16 16 4"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[16, 16, 16, 4])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp16")
ap.add_argument("--rounds", type=int, default=5)
a = ap.parse_args()
runs = {}
for name in ("unsplit", "split"):
    ctx = cd.Context(tuple(a.dims), a.nvec)
    if name == "split":
        ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, 8)
        ctx.peer_connect([ctx.peer_handle()])
        ctx.set_transport("peer")
    L = ctx.links_generate(a.prec, scale_log2=-4)
    x, y = ctx.field(a.prec), ctx.field(a.prec)
    x.generate()
    L.apply(y, x)
    torch.cuda.synchronize()
    runs[name] = (ctx, L, x, y)
s = torch.cuda.current_stream()
res = {}
for r in range(a.rounds):
    for name, (ctx, L, x, y) in runs.items():
        for g in ("1", "0"):
            os.environ["CD_RING_GATHER"] = g
            L.apply(y, x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 200
            e0.record(s)
            for i in range(n):
                L.apply(y, x) if i % 2 == 0 else L.apply(x, y)
            e1.record(s)
            torch.cuda.synchronize()
            res.setdefault(f"{name}_gather{g}", []).append(e0.elapsed_time(e1) / n * 1e3)
print(json.dumps({"dims": a.dims, "prec": a.prec, "variant": runs["split"][0].variants(a.prec)[runs["split"][0].chosen_variant(a.prec)],
                  **{k: round(statistics.median(v), 2) for k, v in res.items()}}))
