"""Compressed (5-matrix) vs full (9-matrix) links, one configuration: chained applies under
sustained load for the full ring, the compressed TMA ring and (CD_COMP_RING=0 in a second
process) the fine-grained compressed kernel.   python profiles/run_compressed_ab.py --dims 16 16 16 32 --prec fp16"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402
import perfmodel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[8, 8, 8, 8])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp32")
ap.add_argument("--secs", type=float, default=1.0)
a = ap.parse_args()
dims = tuple(a.dims)
V = dims[0] * dims[1] * dims[2] * dims[3]
ctx = cd.Context(dims, a.nvec)
L = ctx.links_generate(a.prec, kind="hermitian", scale_log2=-4)
C, _ = L.compress_hermitian(check=False)
x, y = ctx.field(a.prec), ctx.field(a.prec)
x.generate()
N = 2 * a.nvec
rec = 4 * N * N + 16 if a.prec == "fp16" else 8 * N * N
vrec = 4 * N + 16 if a.prec == "fp16" else 8 * N
for name, op in (("full", L), ("compressed", C), ("full", L), ("compressed", C)):
    op.apply(y, x)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    tot, n = 0.0, 0
    t_end = time.perf_counter() + a.secs
    while time.perf_counter() < t_end:
        x.generate()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(10):
            op.apply(y, x) if i % 2 == 0 else op.apply(x, y)
        e1.record(s)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
        n += 10
    us = tot / n * 1e3
    hbm = V * ((9 if name == "full" else 5) * rec + 9 * vrec)
    print(json.dumps({"dims": dims, "prec": a.prec, "op": name, "comp_ring": os.environ.get("CD_COMP_RING", "1"),
                      "us": round(us, 2), "TBs_stored_bytes": round(hbm / us / 1e6, 3)}), flush=True)
