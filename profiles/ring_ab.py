"""A/B timing of the ring variants (CUDA graph of K chained applies, best of 5) for the library
named by CD_LIB_PATH.  python profiles/ring_ab.py --dims 8 8 8 8 --prec fp16 --reps 40 --tag after"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import run_apply  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[8, 8, 8, 8])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp16")
ap.add_argument("--reps", type=int, default=40)
ap.add_argument("--tag", default="")
ap.add_argument("--match", default="ring")
a = ap.parse_args()
ctx, L, x, y = run_apply.setup(tuple(a.dims), a.nvec, a.prec)
for i, name in enumerate(ctx.variants(a.prec)):
    if a.match not in name:
        continue
    us = run_apply.time_variant(ctx, L, x, y, i, a.reps, graph=True)
    print(json.dumps({"tag": a.tag, "dims": a.dims, "prec": a.prec, "variant": name, "us": round(us, 2)}), flush=True)
