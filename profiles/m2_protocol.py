"""Why does bench.py's M2 hot time (CUDA graph of 200 chained applies) differ from
run_apply.py --graph (781 chained applies)?  Same variant, several protocols."""
import os
import sys
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

dims, nvec, prec = (4, 4, 4, 4), 24, "fp32"
big = None
if len(sys.argv) > 2:   # allocate (and keep) a large buffer first, like the bench's M5 headline context
    big = torch.empty(int(float(sys.argv[2]) * 2**30), dtype=torch.uint8, device="cuda")
    big.fill_(1)
ctx = cd.Context(dims, nvec)
L = ctx.links_generate(prec, scale_log2=-4)
a, b = ctx.field(prec), ctx.field(prec)
a.generate()
L.apply(b, a)
var = int(sys.argv[1]) if len(sys.argv) > 1 else -1
if var >= 0:
    ctx.set_option(cd.CD_OPT_VARIANT, var)
print("variant", ctx.variants(prec)[ctx.chosen_variant(prec) if var < 0 else var])
torch.cuda.synchronize()


def graph(K, s):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        x, y = a, b
        for _ in range(K):
            L.apply(y, x, s)
            x, y = y, x
    return g


def timed(g, K, s, gen, sleep):
    ts = []
    for _ in range(10):
        with torch.cuda.stream(s):
            if gen:
                a.generate(stream=s)
            if sleep:
                torch.cuda._sleep(200000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / K)
    return statistics.median(ts), min(ts)


for K in (200, 781):
    for sname in ("side",):
        s = torch.cuda.Stream() if sname == "side" else torch.cuda.current_stream()
        g = graph(K, s)
        g.replay()
        torch.cuda.synchronize()
        for gen in (0, 1):
            for sleep in (0, 1):
                med, mn = timed(g, K, s, gen, sleep)
                print(f"K={K} stream={sname} generate={gen} sleep={sleep}: median {med:.3f} us  min {mn:.3f} us", flush=True)
