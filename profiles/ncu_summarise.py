"""Summarise ncu reports (one row per profiled launch) into a CSV: duration, DRAM bytes, DRAM and
L2 throughput, achieved occupancy, registers, tensor-pipe utilisation.
python profiles/ncu_summarise.py out.csv rep1.ncu-rep [rep2.ncu-rep ...]"""
import csv
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"]
rows = []
for rep in sys.argv[2:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = {"report": rep.split("/")[-1], "kernel": row[h.index("Kernel Name")][:60]}
        for m in M:
            if m in h:
                d[m + " [" + units[h.index(m)] + "]"] = row[h.index(m)]
        rows.append(d)
keys = []
for d in rows:
    keys += [k for k in d if k not in keys]
with open(sys.argv[1], "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=keys)
    w.writeheader()
    w.writerows(rows)
for d in rows:
    print(d)
