"""Which factor makes bench.measure_config's M2 graph slower than m2_protocol's?"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

flush_first = int(sys.argv[1])
capture_in_ctx = int(sys.argv[2])
tune = int(sys.argv[3])
dims, nvec, prec = (4, 4, 4, 4), 24, "fp32"
ctx = cd.Context(dims, nvec)
L = ctx.links_generate(prec, kind="general", scale_log2=-4)
a, b = ctx.field(prec), ctx.field(prec)
a.generate()
if not tune:
    ctx.set_option(cd.CD_OPT_VARIANT, 5)
L.apply(b, a)
if flush_first:
    ctx.flush_l2(256 << 20)
torch.cuda.synchronize()
K = 200
s = torch.cuda.Stream()


def cap():
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        x, y = a, b
        for _ in range(K):
            L.apply(y, x, s)
            x, y = y, x
    return g


if capture_in_ctx:
    with torch.cuda.stream(s):
        g = cap()
else:
    g = cap()
ts = []
with torch.cuda.stream(s):
    for _ in range(20):
        a.generate(stream=s)
        torch.cuda._sleep(200000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / K)
print(f"flush_first={flush_first} capture_in_ctx={capture_in_ctx} tune={tune} "
      f"variant={ctx.variants(prec)[ctx.chosen_variant(prec) if tune else 5]}: median {statistics.median(ts):.3f} us")
