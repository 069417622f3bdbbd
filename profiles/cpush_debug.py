"""Debug driver: chain variant (argv[5], default 4000) on small lattices, n = 1..4 (run under compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1612_07873_b200 as cd
dims = tuple(int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (2, 2, 2, 2)
for n in (1, 2, 3, 4):
    ctx = cd.Context(dims, 24)
    ctx.set_option(cd.CD_OPT_VARIANT, int(sys.argv[5]) if len(sys.argv) > 5 else 4000)
    L = ctx.links_generate("fp32", scale_log2=-4)
    x, y = ctx.field("fp32"), ctx.field("fp32")
    x.generate()
    try:
        L.apply_chain(x, y, n)
        print("n", n, "ok", float(np.linalg.norm(y.export())), flush=True)
    except cd.CDError as e:
        print("n", n, "error", e, flush=True)
        break
