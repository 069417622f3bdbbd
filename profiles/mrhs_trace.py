"""Analyse the CTA-0 event trace of the tcgen05 multi-RHS kernel (diagnostic).

    CD_MRHS_TRACE=gpurun_out/tr.bin python profiles/run_mrhs.py --reps 1
    python profiles/mrhs_trace.py gpurun_out/tr.bin

Events (clock64 per hop h / item t): 0 producer issued hop h, 1 MMA saw A of hop h, 2 MMA saw B of
hop h, 3 builder got a free B slot, 4 builder saw the link record, 5 builder published B, 6-8
epilogue start / accumulator ready / stored, 9 MMA started item t, 10 producer got a free stage for hop h."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(12, 512)
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
# recycle latencies (NBS B slots, S ring stages; argv[2], argv[3], default 3 and 5)
NBS = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S = int(sys.argv[3]) if len(sys.argv) > 3 else 5
print(f"B published -> MMA sees B          {np.mean(t[2, H] - t[5, H]):8.0f}")
print(f"MMA sees B(h) -> builder slot h+{NBS}  {np.mean(t[3, H + NBS] - t[2, H]):8.0f}   (MMA exec + commit + wake)")
print(f"MMA sees B(h) -> producer h+{S}     {np.mean(t[0, H + S] - t[2, H]):8.0f}   (MMA exec + commit + reissue)")
print(f"MMA: B(h) -> A(h+1) seen          {np.mean(t[1, H + 1] - t[2, H]):8.0f}")
print(f"producer: issued h -> stage h+1   {np.mean(t[10, H + 1] - t[0, H]):8.0f}   (waiting for a free stage)")
print(f"producer: stage -> copies issued  {np.mean(t[0, H] - t[10, H]):8.0f}")
