"""Analyse the CTA-0 event trace of the tcgen05 multi-RHS kernel (diagnostic).

    CD_MRHS_TRACE=gpurun_out/tr.bin python profiles/run_mrhs.py --reps 1
    python profiles/mrhs_trace.py gpurun_out/tr.bin

Events (clock64 per hop h / item t): 0 producer issued hop h, 1 MMA saw A of hop h, 2 MMA saw B of
hop h, 3 builder got a free B slot, 4 builder saw the link record, 5 builder published B, 6-8
epilogue start / accumulator ready / stored, 9 MMA started item t."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(10, 512)
H = np.arange(18, min(230, int((t[2] > 0).sum()) - 1))
I = np.arange(3, min(25, int((t[9] > 0).sum()) - 1))


def d(a, b):
    return float(np.mean(t[a, H] - t[b, H]))


print(f"hop period (cycles)               {np.mean(np.diff(t[2, H])):8.0f}")
print(f"producer issue -> MMA sees A      {d(1, 0):8.0f}   (TMA latency incl. ring back-pressure)")
print(f"MMA waits for B after A           {d(2, 1):8.0f}")
print(f"builder: slot -> link record      {d(4, 3):8.0f}")
print(f"builder: link record -> B ready   {d(5, 4):8.0f}")
print(f"item period                       {np.mean(np.diff(t[9, I])):8.0f}")
print(f"epilogue wait / work              {np.mean(t[7, I] - t[6, I]):8.0f} / {np.mean(t[8, I] - t[7, I]):.0f}")
