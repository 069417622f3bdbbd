"""Is the 2^4 chain's time data dependent?  Times variant --variant over n applies per launch for
(a) a finite start vector (re-imported before every launch), (b) a start vector scaled so the
iterate overflows to inf/NaN within a few applies, (c) an all-zero vector; nvidia-smi SM clock
sampled around each case.  python profiles/chain_data_dep.py --variant 4000 --n 800"""
import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", type=int, default=4000)
ap.add_argument("--n", type=int, default=800)
ap.add_argument("--reps", type=int, default=9)
a = ap.parse_args()
dims, nvec = (2, 2, 2, 2), 24
ctx = cd.Context(dims, nvec)
ctx.set_option(cd.CD_OPT_VARIANT, a.variant)
L = ctx.links_upload(synth.links(dims, 2 * nvec, kind="general", scale_log2=-4), "fp32")
x, y = ctx.field("fp32"), ctx.field("fp32")
v = synth.vector(dims, 2 * nvec)
cases = {"finite": v, "overflowing": v * 1e37, "zero": np.zeros_like(v)}


def clock():
    try:
        return int(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                                  capture_output=True, text=True).stdout.strip().split()[0])
    except Exception:
        return -1


for rnd in range(2):
    for name, v0 in cases.items():
        ts = []
        for _ in range(a.reps):
            x.import_(v0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.apply_chain(x, y, a.n)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / a.n)
        fin = bool(np.isfinite(x.export()).all())
        print(json.dumps({"round": rnd, "case": name, "variant": a.variant, "n": a.n, "us_med": round(float(np.median(ts)), 4),
                          "us_min": round(min(ts), 4), "final_finite": fin, "sm_mhz_after": clock()}), flush=True)
