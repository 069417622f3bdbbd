"""Split (self-halo, peer transport) vs unsplit M5 applies under sustained load, alternating
windows, with the unsplit run also without PDL -- separates the halo cost from the PDL overlap
the unsplit chain gets.   python profiles/split_sustained.py [--mask 8] [--secs 1.0] [--rounds 3]"""
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

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[16, 16, 16, 32])
ap.add_argument("--nvec", type=int, default=24)
ap.add_argument("--prec", default="fp16")
ap.add_argument("--mask", type=int, default=8)
ap.add_argument("--variant", type=int, default=10)
ap.add_argument("--secs", type=float, default=1.0)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--nccl-reserve", type=int, nargs="*", default=[],
                help="also time the (unfused) NCCL split with these SM reserves")
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
runs = {}
runs_wanted = ["unsplit", "unsplit_nopdl", "split_peer", "split_peer_unfused"] + \
    [f"split_nccl_r{r}" for r in a.nccl_reserve]
for name in runs_wanted:
    os.environ["CD_FUSE_SPLIT"] = "0" if name == "split_peer_unfused" else "1"   # read at context creation
    ctx = cd.Context(dims, a.nvec)
    if name.startswith("split_peer"):
        ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, a.mask)
        ctx.peer_connect([ctx.peer_handle()])
        ctx.set_transport("peer")
    if name.startswith("split_nccl"):
        ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, a.mask)
        ctx.set_transport("nccl")
        ctx.set_option(cd.CD_OPT_NCCL_SM_RESERVE, int(name.split("_r")[1]))
    if name == "unsplit_nopdl":
        ctx.set_option(cd.CD_OPT_PDL, 0)
    ctx.set_option(cd.CD_OPT_VARIANT, a.variant)
    L = ctx.links_generate(a.prec, scale_log2=-4)
    x, y = ctx.field(a.prec), ctx.field(a.prec)
    x.generate()
    runs[name] = (ctx, L, x, y)
for r in range(a.rounds):
    for name, (ctx, L, x, y) in runs.items():
        t_end = time.perf_counter() + a.secs
        s = torch.cuda.current_stream()
        tot, n = 0.0, 0
        t0 = time.perf_counter()
        while time.perf_counter() < t_end:
            x.generate()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for i in range(16):
                L.apply(y, x) if i % 2 == 0 else L.apply(x, y)
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
            n += 16
        t1 = time.perf_counter()
        cl = [c for (t, c, p) in rows if t0 <= t <= t1]
        print(json.dumps({"round": r, "run": name, "us": round(tot / n * 1e3, 2),
                          "sm_mhz": statistics.median(cl) if cl else None}), flush=True)
proc.terminate()
