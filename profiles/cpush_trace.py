"""Summarise a CD_CHAIN_TRACE dump of the cluster push chain (variant 4000): median cycles of each
event relative to warp 0's start of the same apply, over applies 100..999.
python profiles/cpush_trace.py trace.bin"""
import sys

import numpy as np

tr = np.fromfile(sys.argv[1], dtype=np.int64).reshape(40, 1024)
ts = np.arange(100, 1000)
base = tr[0, ts]
names = {}
for w in range(8):
    for e, nm in enumerate(("start", "X record landed", "math done", "pushed")):
        names[4 * w + e] = f"w{w} {nm}"
    names[32 + w] = f"w{w} remote landed"
print(f"period (w0 start -> next start): {np.median(tr[0, ts + 1] - base):.0f} cycles")
for r, nm in sorted(names.items(), key=lambda kv: (kv[0] % 32 // 4 if kv[0] < 32 else kv[0] - 32, kv[0] >= 32 and 1.5 or kv[0] % 4)):
    d = tr[r, ts] - base
    print(f"{nm:22s} {np.median(d):8.0f}  (p10 {np.percentile(d, 10):.0f}, p90 {np.percentile(d, 90):.0f})")
print(f"prologue: entry -> after cluster barrier {tr[38, 0] - tr[39, 0]} cycles, -> apply 0 start {tr[0, 0] - tr[39, 0]}, "
      f"apply 1 start {tr[0, 1] - tr[39, 0]}, apply 2 start {tr[0, 2] - tr[39, 0]}")
