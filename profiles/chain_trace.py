"""Analyse the CTA-0 clock64 trace of the LL-register chain (CD_CHAIN_TRACE).
Absolute clock64 per apply t: row 4*wk+e for hop warp wk (e: 0 start, 1 record landed,
2 passed (warp 0) / arrived at (hop warps) the partials barrier); warp 0 also 36 summed the
partials, 37 issued the LL store, 38 arrived at the go barrier, 39 wrote its trace.
Times are printed relative to warp 0's start of the same apply."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(40, 1024).astype(np.float64)
T = np.arange(50, 1000)
s0 = t[0, T]


def q(x):
    return f"{np.median(x):7.0f} (p10 {np.percentile(x, 10):6.0f}, p90 {np.percentile(x, 90):6.0f})"


print(f"period (warp 0)                {q(np.diff(t[0, T]))}")
print(f"warp 0 X-term record lands     {q(t[1, T] - s0)}")
print(f"warp 0 passed partial barrier  {q(t[2, T] - s0)}")
print(f"warp 0 summed partials         {q(t[36, T] - s0)}")
print(f"warp 0 issued LL store         {q(t[37, T] - s0)}")
print(f"warp 0 arrived at go barrier   {q(t[38, T] - s0)}")
print(f"warp 0 trace written           {q(t[39, T] - s0)}")
for k in range(1, 9):
    print(f"hop warp {k} (SMSP {k % 4}): start {q(t[4 * k, T] - s0)}  landed {q(t[4 * k + 1, T] - s0)}  "
          f"arrived {q(t[4 * k + 2, T] - s0)}")
