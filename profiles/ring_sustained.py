"""Variant timing under SUSTAINED load (power-capped clocks): cycle through kernel variants, each
for --secs seconds of chained applies, --rounds times, and print per window the time per apply
and the median SM clock (nvidia-smi -lms 20).  Short tuning bursts run at full clock; the bench's
timed region runs power-capped, where variants rank differently.

    python profiles/ring_sustained.py --dims 16 16 16 32 --nvec 24 --prec fp16 --variants 9 10 1 2 --secs 0.4
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402
import perfmodel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[16, 16, 16, 32])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp16")
ap.add_argument("--variants", type=int, nargs="+", required=True)
ap.add_argument("--secs", type=float, default=0.4)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()

rows = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-i", "0",
                         "-lms", "20"], stdout=subprocess.PIPE, text=True)


def reader():
    for line in proc.stdout:
        p = [x.strip() for x in line.split(",")]
        try:
            rows.append((time.perf_counter(), float(p[0]), float(p[1])))
        except ValueError:
            pass


threading.Thread(target=reader, daemon=True).start()
dims = tuple(a.dims)
V = dims[0] * dims[1] * dims[2] * dims[3]
ctx = cd.Context(dims, a.nvec)
L = ctx.links_generate(a.prec, scale_log2=-4)
x, y = ctx.field(a.prec), ctx.field(a.prec)
x.generate()
names = ctx.variants(a.prec)
mb = perfmodel.metric_bytes_per_site(a.nvec, a.prec) * V
out = []
for r in range(a.rounds):
    for var in a.variants:
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        L.apply(y, x)
        torch.cuda.synchronize()
        t_end = time.perf_counter() + a.secs
        s = torch.cuda.current_stream()
        tot_ms, n = 0.0, 0
        t0 = time.perf_counter()
        while time.perf_counter() < t_end:
            x.generate()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            k = 20
            for i in range(k):
                L.apply(y, x) if i % 2 == 0 else L.apply(x, y)
            e1.record(s)
            torch.cuda.synchronize()
            tot_ms += e0.elapsed_time(e1)
            n += k
        t1 = time.perf_counter()
        cl = [c for (t, c, p) in rows if t0 <= t <= t1]
        pw = [p for (t, c, p) in rows if t0 <= t <= t1]
        us = tot_ms / n * 1e3
        rec = {"round": r, "variant": names[var], "us": round(us, 2), "TBs": round(mb / us / 1e6, 3),
               "pct8": round(100 * mb / us / 1e3 / 8000, 1),
               "sm_mhz": statistics.median(cl) if cl else None, "power_w": statistics.median(pw) if pw else None}
        out.append(rec)
        print(json.dumps(rec), flush=True)
proc.terminate()
if a.json:
    with open(a.json, "a") as f:
        for rec in out:
            f.write(json.dumps(dict(rec, dims=dims, nvec=a.nvec, prec=a.prec)) + "\n")
