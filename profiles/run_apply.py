"""Profiling driver: a few chained applies of one configuration with a forced kernel variant.

    python profiles/run_apply.py --dims 8 8 8 8 --nvec 24 --prec fp32 --variant 0 --reps 6 [--dagger]
    python profiles/run_apply.py --sweep [--dims ...]   # time every variant (CUDA events), print a table

Used under `ncu` (launch lists, --set full captures) and for the variant sweep tables in
profiles/.  Links/vectors come from the device generator (bench recipe, links x 2^-4).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402
import perfmodel  # noqa: E402


def setup(dims, nvec, prec):
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate(prec, kind="general", scale_log2=-4)
    a, b = ctx.field(prec), ctx.field(prec)
    a.generate()
    torch.cuda.synchronize()
    return ctx, L, a, b


def time_variant(ctx, L, a, b, var, reps, dagger=False, flush=False, graph=False, chain=False):
    ctx.set_option(cd.CD_OPT_VARIANT, var)
    f = L.apply_dagger if dagger else L.apply
    if chain:   # one persistent kernel for all reps applies
        try:
            L.apply_chain(a, b, 4, dagger)
        except cd.CDError:
            return float("nan")
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            L.apply_chain(a, b, reps, dagger)
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps * 1e3)
        return best
    for _ in range(3):
        f(b, a)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    if graph:   # K chained applies captured in one CUDA graph (no host launch overhead)
        gs = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            x, y = a, b
            for _ in range(reps):
                f(y, x, gs)
                x, y = y, x
        g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps * 1e3)
        return best
    if not flush:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        x, y = a, b
        for _ in range(reps):
            f(y, x)
            x, y = y, x
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    ts = []
    for _ in range(reps):
        ctx.flush_l2(512 << 20)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        f(b, a)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=4, default=[8, 8, 8, 8])
    ap.add_argument("--nvec", type=int, default=24)
    ap.add_argument("--prec", default="fp32")
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--dagger", action="store_true")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--cold", action="store_true", help="L2 flush before every timed apply")
    ap.add_argument("--graph", action="store_true", help="time K chained applies replayed as one CUDA graph")
    ap.add_argument("--chain", action="store_true", help="time coarse_dslash_apply_chain (one persistent kernel)")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    dims = tuple(a.dims)
    ctx, L, x, y = setup(dims, a.nvec, a.prec)
    V = dims[0] * dims[1] * dims[2] * dims[3]
    mb = perfmodel.metric_bytes_per_site(a.nvec, a.prec) * V
    fl = perfmodel.flops_per_site(a.nvec) * V
    if not a.sweep:
        ctx.set_option(cd.CD_OPT_VARIANT, a.variant)
        f = L.apply_dagger if a.dagger else L.apply
        for _ in range(a.reps):
            f(y, x)
            x, y = y, x
        torch.cuda.synchronize()
        print("variant", ctx.variants(a.prec)[ctx.chosen_variant(a.prec, a.dagger)] if a.variant < 0
              else ctx.variants(a.prec)[a.variant])
        return
    rows = []
    cands = list(enumerate(ctx.variants(a.prec)))
    if a.chain:
        cands = [(1000, f"cluster_chain_{a.prec}_nv{a.nvec}")] + \
            [(2000 + i, "ll_" + nm) for i, nm in cands] + cands
    for var, name in cands:
        reps = max(20, min(2000, int(2e5 / max(1, V))))
        us = time_variant(ctx, L, x, y, var, reps, a.dagger, a.cold, a.graph, a.chain)
        rows.append({"variant": name, "us": round(us, 3), "GBs": round(mb / us / 1e3, 1),
                     "GFLOPS": round(fl / us / 1e3, 1), "pct_8TBs": round(100 * mb / us / 1e3 / 8000, 1)})
        print(f"{'x'.join(map(str, dims))} nvec={a.nvec} {a.prec} {'cold' if a.cold else ('graph' if a.graph else ('chain' if a.chain else 'hot'))} "
              f"{name:28s} {us:9.3f} us  {mb / us / 1e3:8.1f} GB/s  {fl / us / 1e3:8.1f} GFLOPS", flush=True)
    if a.json:
        with open(a.json, "a") as fh:
            fh.write(json.dumps({"dims": dims, "nvec": a.nvec, "prec": a.prec, "cold": a.cold, "graph": a.graph, "chain": a.chain,
                                 "dagger": a.dagger, "rows": rows}) + "\n")


if __name__ == "__main__":
    main()
